#!/bin/bash
# ncu --set full capture of the assembly kernel (config 4, one launch) of the
# build PHFEM_LIB points at (default lib/); output gpurun_out/asm_${1:-new}
C="python bench.py --steps 1 --warmup 1 --no-solve --no-cpu"
$C > gpurun_out/plain_${1:-new}.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:assemble_k -s 1 -c 1 -o gpurun_out/asm_${1:-new} $C > gpurun_out/ncu_${1:-new}.log 2>&1
