#!/usr/bin/env python
"""Benchmark of the phfem B200 hot path (BASELINE.json metric:
"tets/s refine+connect+assemble+condense (fp64); Schur solve s; % HBM peak").

Workload (default): config 4, the 128^3 x 6 Kuhn mesh (12,582,912 tets,
Dirichlet z=0, u = sin sin sin, reference operator c=1).  One step = one
pass of the hot path over that device-resident mesh: edge + face
connectivity (bit-exact reference numbering), fused assembly + element-local
Schur condensation into the SELL face matrix, and one 12-way red refinement
of the mesh (12.6M -> 151M tets).  `value` is tets of the input mesh per
second over the whole job; the Schur solve (Jacobi-PCG to the reference's
stopping rule) is timed once after the steps and reported as `schur_solve`.

Arms:
  python bench.py [--gpus N --steps K --warmup W]      this repo (CUDA)
  python bench.py --impl reference ...                  the reference's own CPU
       implementation (oracle/_ref: /root/reference/proj/src compiled by
       oracle/Makefile) on a bounded Kuhn sample, rank 0 only.
Multi-GPU: one process per GPU (torchrun); the path does not shard
(replicas only), so every rank runs an independent replica and
the job time is the max over ranks (scaling "weak").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "tets/s refine+connect+assemble+condense (fp64); Schur solve s; % HBM peak"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """SM clocks + throttle reasons during the timed region: NVML polled
    every 2 ms from a thread (a sample on entry and one on exit, so even a
    short region is covered), nvidia-smi as the fallback."""

    # NVML clocks-event reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, reason_bits)
        self.stop = threading.Event()
        self.nv = None
        self.h = None

    def _handle(self):
        import pynvml as nv
        import torch

        nv.nvmlInit()
        self.nv = nv
        try:
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            self.h = nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)

    def _sample(self):
        nv = self.nv
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                          nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM), int(r)))

    def _loop(self):
        while not self.stop.wait(0.002):
            self._sample()

    def __enter__(self):
        try:
            self._handle()
            self._sample()
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def __exit__(self, *a):
        if self.nv is not None:
            self.stop.set()
            self.t.join(timeout=2)
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({n for _, _, r in self.rows for n, bit in self.BITS.items() if r & bit})
        return {"sm_mhz": statistics.median(x[0] for x in self.rows), "sm_max_mhz": max(x[1] for x in self.rows),
                "reasons": reasons, "samples": len(self.rows), "source": "nvml"}


# ---------------------------------------------------- algorithmic bytes


def ncu_facts():
    """Per-kernel facts extracted from the committed ncu --set full captures
    (tools/ncu_to_json.py -> profiles/ncu_kernels.json)."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_kernels.json")
    try:
        with open(p) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def algorithmic_bytes(nc, ne, ned, nf, nb, nnz_s, l, k_coef=0, elem=True):
    """compulsory bytes per stage (int32 ids, fp64 reals,
    int8 sigma, u8 class, int64 row pointers, int32 columns).  The step's
    condensed S is element-major (elem: 10 fp64 S_T values + 4 int32 rows
    per element and the assembled diagonal) or SELL rows (12 nnz_s).  The CG
    on the element-major S (the pipeline's system) reads per row its two
    slots and the diagonal (16 l) and per element the six off-diagonal
    S_T values and four row ids (64 ne); the vectors: p and q in the SpMV
    (16 l), r, q, d read and r written in the update (32 l), x, p, r, d
    read and x, p written in the direction update (48 l)."""
    b_edges = 44 * ne + 8 * ned
    b_faces = 60 * ne + 24 * nc + 12 * nb + 33 * nf
    s_out = 96 * ne + 8 * l if elem else 12 * nnz_s
    b_asm = 36 * ne + 24 * nc + 13 * nf + k_coef * ne + s_out + 16 * l + 8
    b_refine = 260 * ne + 48 * nc + 24 * ned + 72 * nb
    b_cg = (64 * ne + 16 * l if elem else 12 * nnz_s) + 96 * l
    return dict(connect=b_edges + b_faces, assemble=b_asm, refine=b_refine, refine_boundary=72 * nb,
                cg_iteration=b_cg)


# ---------------------------------------------------------- reference arm


def reference_sample(n: int):
    from oracle_bind import Oracle, RefCtx, ref_available

    if not ref_available():
        raise RuntimeError("oracle/_ref/libphfem_ref.so not built")
    O = Oracle()
    m = O.kuhn(n, n, n, dmask=0x10)
    return m, RefCtx


def reference_step(m, RefCtx, workers):
    t0 = time.perf_counter()
    r = RefCtx(m)
    t = r.connectivity()
    r.assemble(3)
    r.build_schur(workers)
    r.refine()
    return time.perf_counter() - t0, t


def run_reference(args, rank):
    if rank != 0:
        return
    # config-3-sized samples (64^3 x 6, ~15-20 s a step on 8-16 host cores)
    # while the whole run stays within a few minutes, smaller ones otherwise
    n = args.ref_n or (64 if args.steps + args.warmup <= 10 else (48 if args.steps + args.warmup <= 20 else 32))
    cores = os.cpu_count() or 1
    m, RefCtx = reference_sample(n)
    for _ in range(args.warmup):
        reference_step(m, RefCtx, cores)
    times = [reference_step(m, RefCtx, cores)[0] for _ in range(args.steps)]
    sec = sum(times) / len(times)
    value = m.ne / sec
    sample = (f"Kuhn {n}^3 x 6 = {m.ne} tets (config-4 shape and problem at reduced n): num_edges, "
              f"edge_pairs_to_elems, faces_up, full_face_table, assemble_system, build_schur(workers={cores}), "
              f"red_refine per step")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tets/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg4-shape Kuhn {n}^3 (bounded CPU sample)", "mesh_tets": m.ne},
            "cpu_baseline": {"value": value, "unit": "tets/s", "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "tets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(n=64, gpu_iterations=None, l_target=None):
    """Reference CPU path (oracle/_ref) on a bounded sample of the workload,
    stage by stage: connectivity, assemble_system,
    build_schur(nproc) and build_schur(1), red_refine, and a 200-iteration
    prefix of pcg_jacobi for the per-iteration cost."""
    try:
        m, RefCtx = reference_sample(n)
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unit": "tets/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}
    cores = os.cpu_count() or 1
    r = RefCtx(m)
    t0 = time.perf_counter()
    r.connectivity()
    t1 = time.perf_counter()
    r.assemble(3)
    t2 = time.perf_counter()
    r.build_schur(cores)
    t3 = time.perf_counter()
    r.refine()
    t4 = time.perf_counter()
    sec = t4 - t0
    r2 = RefCtx(m)
    r2.connectivity()
    r2.assemble(3)
    t5 = time.perf_counter()
    r2.build_schur(1)
    t6 = time.perf_counter()
    cg_iters = 200
    cg_s, _ = r2.cg_prefix(cg_iters)
    l_sample = r2.counts()["l"]
    out = {"value": m.ne / sec, "unit": "tets/s", "cores": cores, "kind": "reference",
           "sample": (f"Kuhn {n}^3 x 6 = {m.ne} tets, one pass of num_edges + edge_pairs_to_elems + faces_up + "
                      f"full_face_table + assemble_system + build_schur(workers={cores}) + red_refine in {sec:.2f} s; "
                      f"only build_schur uses more than one thread"),
           "stages_s": {"connectivity": t1 - t0, "assemble_system": t2 - t1, f"build_schur_{cores}": t3 - t2,
                        "build_schur_1": t6 - t5, "red_refine": t4 - t3},
           "cg_s_per_iteration": cg_s / cg_iters, "cg_sample_l": l_sample}
    if gpu_iterations and l_target:
        # labelled estimate: per-iteration cost scaled by L,
        # times the GPU-measured iteration count of the full problem
        out["cg_full_estimate_s"] = cg_s / cg_iters * (l_target / l_sample) * gpu_iterations
    return out


def measure_fp64_peak(ph, torch, stream, iters=16384, reps=5):
    """fp64 FMA throughput of this GPU (TFLOP/s, best of reps) from the
    library's DFMA probe kernel, timed with CUDA events on its stream."""
    import ctypes

    fn = ph.lib().phfem_gpu_fp64_peak
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    flops = ctypes.c_double()
    best = 0.0
    for _ in range(reps + 1):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn(iters, sink.data_ptr(), None, None, ctypes.byref(flops), stream.cuda_stream)
        e1.record(stream)
        e1.synchronize()
        best = max(best, flops.value / (e0.elapsed_time(e1) / 1e3) / 1e12)
    return best


# ------------------------------------------------------- multi-process


def dist_setup(world: int, local: int, backend: str = "nccl"):
    """One process per GPU (torchrun env): the process group, or None at
    world size 1.  NCCL carries only the barrier and the max-over-ranks
    timing; the replicas exchange no data."""
    if world <= 1:
        return None
    import torch
    import torch.distributed as dist

    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return dist


def max_over_ranks(dist, x: float, device=None) -> float:
    """The slowest rank's time (every rank gets it)."""
    if dist is None:
        return float(x)
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(world: int, units_per_rank: int, ms_max: float) -> float:
    """Whole-job units/s: every rank processes the same units (weak scaling)
    and the job takes as long as its slowest rank."""
    return world * units_per_rank / (ms_max / 1e3)


# ------------------------------------------------------------------ ours


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-n", type=int, default=0, help="reference-arm sample n (n^3 x 6 tets); 0: by budget")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch

    torch.cuda.set_device(local)
    dist = dist_setup(world, local)

    import numpy as np

    from paper_2509_11133_b200 import configs
    from paper_2509_11133_b200 import phfem as ph

    cfg = configs.CONFIGS[args.config]
    if args.config == 2:
        run_config2(args, ph, torch, rank)
        return
    mesh = cfg.build()
    nc, ne, nd, nn = mesh.sizes()
    stream = torch.cuda.ExternalStream(ph.stream_ptr())
    launches = ph.lib().phfem_gpu_launch_count
    launches.restype = __import__("ctypes").c_longlong

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    # nnz(S) from an exported (row-form) system first: the warm-up passes
    # then leave the pipeline's element-major system in place
    nnz_s = int(mesh.assemble(cfg.problem)["s_col"].size) if ne <= 2_000_000 else None
    for _ in range(args.warmup):
        stages, counts = mesh.pipeline(cfg.problem, True)
    ned, nf, l, sell_slots, ne_child = (int(v) for v in counts)
    conn = mesh.connectivity()
    sysz = np.zeros(3, dtype=np.int64)

    barrier()
    l0 = launches()
    acc = {}
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            st, _ = mesh.pipeline(cfg.problem, True)
            for k, v in st.items():
                acc[k] = acc.get(k, 0.0) + v
        e1.record(stream)
        e1.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    nlaunch = launches() - l0
    stage_ms = {k: v / args.steps for k, v in acc.items()}
    # the library's rule (capi.cpp: fused_refine_enabled): a pass that both
    # assembles and refines writes the children from the assembly kernel
    fused_refine = os.environ.get("PHFEM_FUSED_REFINE", "1")[:1] != "0"
    ms_max = max_over_ranks(dist, ms, "cuda")
    value = job_throughput(world, ne, ms_max)

    # nnz(S) (true, without SELL padding) from the row structure: every
    # multiplier row has 1 + the non-Neumann other faces of its 1-2 elements
    if nnz_s is None:
        nnz_s = mesh_nnz_s(mesh, cfg.problem)
    hbm, hbm_kind = peaks()
    k_coef = 8 if cfg.coef == "log_uniform" else (24 if cfg.coef == "aniso" else 0)
    B = algorithmic_bytes(nc, ne, ned, nf, nd + nn, nnz_s, l, k_coef)
    conn_ms = stage_ms["star"] + stage_ms["groups"] + stage_ms["number"] + stage_ms["classify"]
    per_stage = {
        "connect": {"ms": conn_ms, "bytes": B["connect"]},
        "assemble_condense": {"ms": stage_ms["assemble"], "bytes": B["assemble"]},
        "refine": {"ms": stage_ms["refine"], "bytes": B["refine"]},
    }
    if fused_refine:
        # the assembly kernel writes the children and new nodes itself
        # (assemble.cu: refine_elem): its bytes are both stages' less the
        # element rows and vertex coordinates read once instead of twice;
        # the refinement stage is the boundary lists alone
        b_fused = B["assemble"] + B["refine"] - B["refine_boundary"] - 16 * ne - 24 * nc
        per_stage["assemble_condense"]["bytes"] = b_fused
        per_stage["refine"]["bytes"] = B["refine_boundary"]
    for k, v in per_stage.items():
        v["gbs"] = v["bytes"] / (v["ms"] / 1e3) / 1e9
        v["hbm_frac"] = v["gbs"] / hbm
        v["tets_per_s"] = ne / (v["ms"] / 1e3)
    # the roofline kernel: the fused assembly kernel whenever the step
    # assembles (the top kernel of every assembling config's launch list,
    # profiles/r2_*_launches_summary.txt), else the longest stage
    dom_name = ("assemble_condense" if stage_ms.get("assemble_kernel", 0.0) > 0
                else max(per_stage, key=lambda k: per_stage[k]["ms"]))
    dom = per_stage[dom_name]
    total_bytes = sum(v["bytes"] for v in per_stage.values())
    step_gbs = total_bytes / (ms / 1e3) / 1e9
    # the dominant kernel's roofline.  The fused assembly kernel is fp64-pipe
    # bound (ncu: sm__pipe_fp64_cycles_active), so its roofline is the fp64
    # one: SASS fp64 flop per launch (committed ncu capture of the same
    # config) over the live kernel time, against the DFMA peak measured on
    # this GPU (MEASURED_PEAKS.json carries no fp64 figure); its HBM
    # fraction is reported beside it.
    roofline = {"bound": "hbm", "achieved": dom["gbs"], "peak": hbm, "unit": "GB/s", "frac": dom["gbs"] / hbm,
                "traffic": None, "kernel": dom_name, "peak_kind": hbm_kind,
                "step": {"algorithmic_bytes": total_bytes, "achieved_gbs": step_gbs, "hbm_frac": step_gbs / hbm,
                         "target_frac": 0.60, "target_ms": total_bytes / (0.60 * hbm * 1e9) * 1e3,
                         "note": "refine + connect + assemble/condense step against the north-star 60% of HBM"}}
    kern_ms = stage_ms.get("assemble_kernel", 0.0)
    # the pipeline's instance: element-major condensed operator (ELEM = 1)
    kname = f"assemble_k<{cfg.problem}, 1>"
    prof = ncu_facts().get(kname) if dom_name == "assemble_condense" else None
    if dom_name == "assemble_condense" and kern_ms > 0:
        b_kern = per_stage["assemble_condense"]["bytes"]
        a_gbs = b_kern / (kern_ms / 1e3) / 1e9
        roofline.update({"kernel": kname, "kernel_ms": kern_ms, "algorithmic_bytes": b_kern,
                         "fused_refinement": fused_refine,
                         "hbm": {"achieved": a_gbs, "peak": hbm, "unit": "GB/s", "frac": a_gbs / hbm,
                                 "peak_kind": hbm_kind}})
        if prof:
            roofline["traffic"] = prof["dram_bytes"]
            roofline["profile"] = prof["source"]
            roofline["fp64_pipe_busy"] = prof["fp64_pipe_frac"]
            if prof.get("fp64_flop") and prof.get("config", cfg.name) == cfg.name:
                roofline.update({"bound": "fp64", "unit": "TFLOP/s", "flop_per_launch": prof["fp64_flop"],
                                 "flop_per_tet": prof["fp64_flop"] / ne,
                                 "achieved": prof["fp64_flop"] / (kern_ms / 1e3) / 1e12})

    # e2e through the public C ABI: pinned host arrays -> device mesh ->
    # pipeline -> counts back
    coords, tets, db, nb = mesh.arrays()
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    hc, ht, hd, hn = pin(coords), pin(tets), pin(db), pin(nb)
    h2d = hc.nbytes + ht.nbytes + hd.nbytes + hn.nbytes
    def e2e_steps(n):
        # double-buffered: step k+1's inputs go up on the copy engine
        # (phfem_mesh_create_from_arrays_async) while step k's pass runs;
        # every step still uploads its whole mesh and reads its counts back
        nxt = ph.Mesh.from_arrays_async(hc, ht, hd, hn)
        cts = None
        for k in range(n):
            cur = nxt
            nxt = ph.Mesh.from_arrays_async(hc, ht, hd, hn) if k + 1 < n else None
            _, cts = cur.pipeline(cfg.problem, True)
            del cur
        return cts

    e2e_steps(args.warmup)  # untimed: lets the device pool reach steady state
    barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    # at least 20 steps: the first step's upload has nothing to overlap with
    # and is charged in full to the timed region
    n_e2e = max(args.steps, 20)
    e2.record(stream)
    t_wall = time.perf_counter()
    cts = e2e_steps(n_e2e)
    e3.record(stream)
    e3.synchronize()
    wall = (time.perf_counter() - t_wall) / n_e2e
    e2e_ms = max(e2.elapsed_time(e3) / n_e2e, wall * 1e3)
    # the PCIe floor of that upload: the same pinned arrays copied alone
    # (no kernels running), device-timed
    dbuf = torch.empty(int(h2d) // 8 + 8, dtype=torch.float64, device="cuda")
    srcs = [torch.from_numpy(a.reshape(-1).view("u1")) for a in (hc, ht, hd, hn)]
    srcs = [a if a.is_pinned() else a.pin_memory() for a in srcs]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dst = dbuf.view(torch.uint8)
    h2d_ms = []
    for _ in range(4):
        ev0.record()
        off = 0
        for a in srcs:
            dst[off:off + a.numel()].copy_(a, non_blocking=True)
            off += a.numel()
        ev1.record()
        ev1.synchronize()
        h2d_ms.append(ev0.elapsed_time(ev1))
    del dbuf
    h2d_alone = min(h2d_ms[1:])
    e2e = {"value": job_throughput(world, ne, max_over_ranks(dist, e2e_ms, "cuda")), "unit": "tets/s",
           "overlap": "double-buffered uploads on the copy engine (create_from_arrays_async); "
                      "the first step's upload is not overlapped",
           "steps": n_e2e, "ms_per_step": e2e_ms,
           "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(cts.nbytes + 7 * 8),
           "h2d_alone_ms": h2d_alone, "h2d_alone_gbs": h2d / (h2d_alone / 1e3) / 1e9,
           "bound": ("PCIe upload" if h2d_alone >= 0.9 * ms_max else "device step"),
           "note": "each step uploads its whole mesh from pinned host memory; the step is bounded by "
                   "max(device step, upload), the upload time measured alone above"}

    # Schur solve (Jacobi-PCG, reference stopping rule), once
    solve = None
    if not args.no_solve:
        # "Schur solve s" = CG + recovery + verify wall time;
        # the CG alone is timed on the device
        # untimed warm-up: a solve capped at a few iterations (its stall is
        # expected) so the timed solve does not pay first-use costs (device
        # pool growth for its vectors, graph instantiation, module loading)
        try:
            mesh.solve_timed(cfg.problem, cfg.tol, max_iter=64)
        except ph.SolverError:
            pass
        r = mesh.solve_timed(cfg.problem, cfg.tol)
        b_it = B["cg_iteration"]
        gbs = b_it / (r["ms_per_iteration"] / 1e3) / 1e9 if r["ms_per_iteration"] else None
        solve = {"seconds": r["total_s"], "cg_seconds": r["cg_ms"] / 1e3, "iterations": r["iterations"],
                 "converged": r["converged"], "accepted_by_verify": r["accepted"], "residual": r["residual"],
                 "ms_per_iteration": r["ms_per_iteration"], "gbs_per_iteration": gbs,
                 "hbm_frac": gbs / hbm if gbs else None, "tol": cfg.tol}
        # verify_solution's three tests (solver.cpp:68-69) with their values
        t = cfg.tol
        checks = {"combined": [r["residual"], t],
                  "primal ||AU-C'L-B||/||B||": [r["r1"] / max(r["norm_rhs"], 1e-300), t],
                  "constraint ||CU-b_D||/(1+||b_D||)": [r["r2"] / (1.0 + r["norm_bd"]), t]}
        solve["verify"] = {k: {"value": float(v), "limit": lim, "pass": bool(v <= lim)} for k, (v, lim) in checks.items()}
        solve["norm_bd"] = r["norm_bd"]
        solve["norm_rhs"] = r["norm_rhs"]
        if not r["accepted"]:
            failed = [k for k, c in solve["verify"].items() if not c["pass"]]
            solve["note"] = (f"verify_solution refuses this converged solve (failed: {', '.join(failed)}; "
                             f"||b_D|| = {r['norm_bd']:.3e}, ||B|| = {r['norm_rhs']:.3e}); the CPU oracle's "
                             f"verdict on the same system is in tests/golden/solution_cfg*.npz (SURVEY finding 8)")

    fp64_peak = measure_fp64_peak(ph, torch, stream)
    if roofline["bound"] == "fp64":
        nominal = 64 * 2 * 148 * 1.965e9 / 1e12
        roofline.update({"peak": fp64_peak, "frac": roofline["achieved"] / fp64_peak,
                         "peak_kind": "measured: DFMA probe kernel on this GPU (phfem_gpu_fp64_peak)",
                         "nominal_peak": nominal, "nominal_frac": roofline["achieved"] / nominal})

    if rank == 0:
        cpu = (cpu_baseline(gpu_iterations=solve["iterations"] if solve else None, l_target=l)
               if (world == 1 and not args.no_cpu) else None)
        line = {
            "metric": METRIC, "value": value, "unit": "tets/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "mesh_tets": ne, "mesh_nodes": nc, "edges": ned, "faces": nf,
                       "multipliers": l, "nnz_S": nnz_s, "children_tets": ne_child, "problem": cfg.problem,
                       "note": cfg.note, "l2": "inputs > L2 (mesh 253 MB; per-step working set several GB)",
                       "parallelism": f"replicas x{world}"},
            "stages_ms": stage_ms, "per_stage": per_stage, "roofline": roofline, "schur_solve": solve,
            "e2e": e2e, "gpu_launches": int(nlaunch), "clocks": clk.summary(), "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_config2(args, ph, torch, rank):
    """Config 2: 1 cube -> 6 Kuhn tets refined level by level up to the first
    level with >= 2e7 tets (level 7, 214,990,848 tets); per level the
    connectivity (edges + faces + classification) and the red refinement that
    produced the next level, device-resident, CUDA-event timed."""
    hbm, hbm_kind = peaks()
    m = ph.Mesh.kuhn(1, 1, 1, dirichlet_mask=0x3F)
    levels = []
    for lv in range(8):
        nc, ne, nd, nn = m.sizes()
        reps = max(1, args.steps if ne < 50_000_000 else 1)
        for _ in range(min(args.warmup, 3) if ne < 50_000_000 else 1):
            m.pipeline(0, do_refine=lv < 7, assemble=False)
        acc = {}
        for _ in range(reps):
            st, cts = m.pipeline(0, do_refine=lv < 7, assemble=False)
            for k, v in st.items():
                acc[k] = acc.get(k, 0.0) + v / reps
        ned, nf = int(cts[0]), int(cts[1])
        conn_ms = acc["star"] + acc["groups"] + acc["number"] + acc["classify"]
        B = algorithmic_bytes(nc, ne, ned, nf, nd + nn, 0, 0)
        row = {"level": lv, "tets": ne, "nodes": nc, "edges": ned, "faces": nf, "connect_ms": conn_ms,
               "connect_tets_per_s": ne / (conn_ms / 1e3), "connect_hbm_frac": B["connect"] / (conn_ms / 1e3) / 1e9 / hbm}
        if lv < 7:
            row.update(refine_ms=acc["refine"], refine_child_tets_per_s=12 * ne / (acc["refine"] / 1e3),
                       refine_hbm_frac=B["refine"] / (acc["refine"] / 1e3) / 1e9 / hbm)
            m.refine()
        levels.append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    top = levels[-1]
    prev = levels[-2]
    step_ms = top["connect_ms"] + prev["refine_ms"]
    if rank == 0:
        print(json.dumps({"metric": "tets/s refine+connect (config 2, level 7)", "value": top["tets"] / (step_ms / 1e3),
                          "unit": "tets/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                          "dtype": "int32/f64", "data": "synthetic",
                          "config": {"workload": "cfg2_cube6_refine", "levels": levels, "peak_kind": hbm_kind}}),
              flush=True)


def mesh_nnz_s(mesh, problem):
    """nnz of S from the face table (rows = multiplier faces)."""
    import numpy as np

    f = mesh.faces()
    fs = f["face_slots"]
    mrow = f["mrow"]
    fos = f["face_of_slot"].reshape(-1, 4)
    nonneu = (mrow[fos] >= 0).sum(axis=1)  # per element
    rows = np.nonzero(mrow >= 0)[0]
    s0 = fs[rows, 0] // 4
    s1 = fs[rows, 1]
    nnz = 1 + (nonneu[s0] - 1)
    inter = s1 >= 0
    nnz = nnz.astype(np.int64)
    nnz[inter] += nonneu[s1[inter] // 4] - 1
    return int(nnz.sum())


if __name__ == "__main__":
    main()
