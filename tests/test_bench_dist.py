"""bench.py's multi-process logic on CPU: world size 2 over gloo (the GPU
runs use NCCL with the same helpers), and the reference arm's rank
behaviour under torchrun (rank 0 alone runs and prints)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, times, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import bench

    dist = bench.dist_setup(world, rank, backend="gloo")
    m = bench.max_over_ranks(dist, times[rank])
    v = bench.job_throughput(world, 1000, m)
    dist.barrier()
    q.put((rank, m, v))
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    times = [10.0, 12.5]
    procs = [ctx.Process(target=_worker, args=(r, 2, port, times, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, m, v in res:
        assert m == 12.5  # the slowest rank's time on every rank
        assert v == pytest.approx(2 * 1000 / 0.0125)  # whole-job units / max time


def test_single_process_helpers():
    sys.path.insert(0, ROOT)
    import bench

    assert bench.dist_setup(1, 0) is None
    assert bench.max_over_ranks(None, 3.5) == 3.5
    assert bench.job_throughput(1, 500, 2.0) == pytest.approx(250000.0)


def _run_bench(env_extra, *args):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=env, cwd=ROOT, timeout=600)


def test_reference_arm_other_ranks_exit_silently():
    r = _run_bench({"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2"}, "--impl", "reference", "--gpus", "2",
                   "--steps", "1", "--warmup", "0")
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


def test_reference_arm_rank0_line():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built")
    r = _run_bench({"RANK": "0", "WORLD_SIZE": "1"}, "--impl", "reference", "--steps", "1", "--warmup", "0",
                   "--ref-n", "4")
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "tets/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
