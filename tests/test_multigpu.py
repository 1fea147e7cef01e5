"""Multi-GPU K3 (include/prg.h prg_k3_pagerank_sharded): the
column-sharded run_kernel3. CPU (gloo, world size 2): the partition rule and
the exchange protocol — disjoint writers combined by all_reduce(SUM) reproduce
the single-writer arrays bit for bit. GPU: world sizes 2 and 3 emulated by host
threads on one device (each "rank" on its own stream; the exchange is done on
the host between SpMVs, kernels never wait on one another) must give ranks and
norm1 bit-identical to the single-GPU timed mode.
"""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O


def _free_port():
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        return sck.getsockname()[1]


def _synthetic_slices(nslices, seed):
    rng = np.random.default_rng(seed)
    # sorted longest first, like the SELL slice list: sizes 32 * (max lane length)
    sizes = np.sort(32 * rng.zipf(1.6, nslices).clip(1, 4096))[::-1]
    sp = np.zeros(nslices + 1, dtype=np.uint32)
    sp[1:] = np.cumsum(sizes)
    return sp


def test_shard_bounds_rule():
    from paper_1603_01876_b200 import capi

    for nslices, world in ((1, 1), (1, 4), (5, 8), (10000, 2), (10000, 3), (70000, 8)):
        sp = _synthetic_slices(nslices, nslices + world)
        b = capi.shard_bounds_host(sp, world)
        assert b[0] == 0 and b[-1] == nslices and np.all(np.diff(b.astype(np.int64)) >= 0)
        total = int(sp[-1])
        for r in range(1, world):  # rank r starts at the first slice at/after r/world of the entries
            want = total * r // world
            assert sp[b[r]] >= want and (b[r] == 0 or sp[b[r] - 1] < want)
    with pytest.raises(capi.PrgError):
        capi.shard_bounds_host(np.array([0, 5, 3], dtype=np.uint32), 2)


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1603_01876_b200 import capi

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sp = _synthetic_slices(20000, 7)
        b = capi.shard_bounds_host(sp, world)
        mine = torch.from_numpy(b.astype(np.int64))
        every = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(every, mine)
        same = all(torch.equal(x, mine) for x in every)
        # exchange protocol: the single-GPU iterate values, split-column part sums and
        # slice sums; each rank writes only what its slices own into a zeroed buffer
        rng = np.random.default_rng(11)
        full = rng.random(32 * 20000) * 1e-7 + rng.integers(0, 2, 32 * 20000) * 1e-300  # incl. subnormal-scale values
        owner = np.repeat(np.searchsorted(b, np.arange(20000), side="right") - 1, 32)
        buf = torch.from_numpy(np.where(owner == rank, full, 0.0))
        capi.torch_allreduce()(buf)
        exact = np.array_equal(buf.numpy().view(np.int64), full.view(np.int64))
        q.put((rank, same, exact))
    finally:
        dist.destroy_process_group()


def test_sharded_exchange_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(same and exact for _, same, exact in res)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("scale,seed,init", [(14, 7, O.GRAPH500), (12, 2, O.UNIFORM)])
def test_k3_sharded_bit_identical(cuda, world, scale, seed, init):
    import threading

    import torch

    from paper_1603_01876_b200 import capi

    n = 1 << scale
    srt = torch.from_numpy(O.k1_sort(O.generate(scale, seed, init), scale)).cuda()
    mat = capi.k2_filter(srt, n, csc=True)
    ref, nref = capi.k3_pagerank(mat, seed=seed, mode=0)
    ref = ref.cpu().numpy()
    bounds = capi.k3_shard_bounds(mat, world)
    assert bounds[0] == 0 and np.all(np.diff(bounds.astype(np.int64)) >= 0)

    barrier = threading.Barrier(world)
    shared = {}

    def host_allreduce(rank):
        def allreduce(buf, strm):
            torch.cuda.ExternalStream(strm).synchronize()  # this rank's SpMV is done
            shared[rank] = buf
            barrier.wait()
            if rank == 0:
                acc = torch.zeros_like(buf)
                for r in range(world):
                    acc += shared[r]
                torch.cuda.synchronize()
                shared["sum"] = acc
            barrier.wait()
            buf.copy_(shared["sum"])
            torch.cuda.synchronize()
            barrier.wait()
        return allreduce

    out = [None] * world
    errors = []

    def run(rank):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                r, norm = capi.k3_pagerank_sharded(mat, rank, world, host_allreduce(rank), seed=seed, stream=st)
            st.synchronize()
            out[rank] = (r.cpu().numpy(), norm)
        except BaseException as e:  # noqa: BLE001
            errors.append(e)
            barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=300)
    assert not errors, errors
    for r, norm in out:
        assert np.array_equal(r.view(np.int64), ref.view(np.int64)) and norm == nref
    mat.close()


def _nccl_world1_worker(port, q):
    import torch
    import torch.distributed as dist

    from paper_1603_01876_b200 import capi

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), PRG_SHARD_EXCHANGE_ALWAYS="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        scale, seed = 14, 7
        n = 1 << scale
        srt = torch.from_numpy(O.k1_sort(O.generate(scale, seed), scale)).cuda()
        mat = capi.k2_filter(srt, n, csc=True)
        ref, nref = capi.k3_pagerank(mat, seed=seed, mode=0)
        st = torch.cuda.Stream()
        inner, calls_box = capi.torch_allreduce(), [0]

        def counted(buf, stream=None):
            calls_box[0] += 1
            inner(buf, stream)

        with torch.cuda.stream(st):
            got, ngot = capi.k3_pagerank_sharded(mat, 0, 1, counted, seed=seed, stream=st)
        st.synchronize()
        same = np.array_equal(got.cpu().numpy().view(np.int64), ref.cpu().numpy().view(np.int64)) and ngot == nref
        calls = calls_box[0]
        mat.close()
        q.put(bool(same) and calls == 20)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_k3_sharded_through_nccl_world1(cuda):
    """The exchange as bench.py --gpus N performs it — capi.torch_allreduce over
    NCCL on the library's stream — on the one GPU this run has (world size 1):
    the callback, the stream ordering and the NCCL call are the real ones."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_world1_worker, args=(_free_port(), q))
    p.start()
    ok = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0 and ok
