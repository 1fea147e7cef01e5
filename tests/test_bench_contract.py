"""CPU: bench.py's formulas and the reference arm's JSON contract.

The reference arm (--impl reference) runs the compiled reference on the host,
so it is exercised here at a tiny scale; the GPU arm is run by the driver.
"""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_algorithmic_bytes_match_survey():
    # S=24, nnz_f = 261,074,939
    n, m, nnz = 1 << 24, 1 << 28, 261074939
    k1, k2, k3, k3_iter = bench.alg_bytes(n, m, nnz, 20)
    assert round(k1 / 1e9, 2) == 8.59
    assert round(k2 / 1e9, 2) == 7.49 or round(k2 / 1e9, 2) == 7.50
    assert round(k3 / 1e9, 1) == 69.5
    assert k3 == 20 * k3_iter + 8 * n


def test_peaks_source():
    peak, src = bench.peaks()
    assert peak > 1000 and isinstance(src, str)


def test_clock_sampler_summary():
    s = bench.ClockSampler(0)
    s.rows = [["0", "1965", "1965", "500", "0x0", "Not Active", "Not Active", "Not Active", "Active"],
              ["0", "1900", "1965", "510", "0x4", "Not Active", "Not Active", "Not Active", "Not Active"]]
    out = s.summary()
    assert out["sm_max_mhz"] == 1965 and out["reasons"] == ["sw_power_cap"] and out["samples"] == 2


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libprpipe_ref.so")),
                    reason="reference library not built")
def test_reference_arm_json_contract():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--scale", "10",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in j
    assert j["impl"] == "reference" and j["value"] > 0
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["d2h_bytes_per_step"] == 0
    assert j["cpu_baseline"]["kind"] == "reference"


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r's stage times: the job's time is the slowest rank's, per entry
        got = bench.max_over_ranks([10.0 + rank, 5.0 - rank, 7.0])
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    """The N>1 bench path (one process per GPU; NCCL on the box) reduces every
    timing to the max over ranks — exercised here with gloo, world size 2."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1] == [11.0, 5.0, 7.0]


def test_whole_job_rate_and_single_process_max():
    assert bench.max_over_ranks([1.5, 2.5]) == [1.5, 2.5]  # no process group: identity
    # value = units all ranks processed / max-over-ranks time (weak scaling)
    assert bench.whole_job_rate(4, 20 * (1 << 28), 0.02) == 4 * 20 * (1 << 28) / 0.02


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libprpipe_ref.so")),
                    reason="reference library not built")
def test_reference_arm_under_torchrun_world2():
    """Launched as the driver does for N>1: rank 0 alone runs the reference
    arm and prints one JSON line; the other rank exits 0 without work."""
    import socket

    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--impl", "reference", "--gpus", "2", "--scale", "8", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["value"] > 0
