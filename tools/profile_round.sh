#!/bin/bash
# The evidence of one round on the GPU box (run through gpurun; one GPU):
#   bench lines of configs 4 (default, with the CPU baseline), 1, 3, 5, the
#   config-2 ladder and the reference arm; the launch list of one config-4
#   step and of 64 CG iterations (ncu, gpu__time_duration + DRAM bytes,
#   --clock-control none); one ncu --set full capture of a config-4 step
#   (all kernels, source-mapped).  Numbers printed under ncu are not bench
#   values: every ncu pass follows a plain run of the same command.
# usage: tools/profile_round.sh TAG   (outputs gpurun_out/TAG_*)
T=${1:-r2}
O=gpurun_out
mkdir -p $O
python bench.py > $O/${T}_cfg4_bench.json 2> $O/${T}_cfg4_bench.err
for c in 1 3 5; do
  python bench.py --config $c --no-cpu > $O/${T}_cfg${c}_bench.json 2> $O/${T}_cfg${c}_bench.err
done
python bench.py --config 2 --steps 3 > $O/${T}_cfg2_bench.json 2> $O/${T}_cfg2_bench.err
python bench.py --impl reference > $O/${T}_reference_arm.json 2> $O/${T}_reference_arm.err
python tools/profile_step.py 4 > $O/${T}_plain_step.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --profile-from-start off --csv --log-file $O/${T}_cfg4_launches.csv python tools/profile_step.py 4 \
      > $O/${T}_ncu_launch.log 2>&1
python tools/cg_probe.py 64 > $O/${T}_plain_cg.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:cg_ --csv --log-file $O/${T}_cfg4_cg_launches.csv python tools/cg_probe.py 64 \
      > $O/${T}_ncu_cg.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -o $O/${T}_step_full \
    python tools/profile_step.py 4 > $O/${T}_ncu_full.log 2>&1
echo done
