"""Multi-rank host logic of the row-group sharding (CPU, gloo, world 2/3).

Each rank computes its groups with the ORACLE (the checker stands in for the
device kernel, which needs a GPU), the ranks all-gather their padded compact
rows with torch.distributed (gloo), and the gathered buffer is un-permuted
through ShardPlan.gathered_row_map; the result must equal the full SpMM bit
for bit.  The CUDA path of the same plan runs in
tests/test_gpu_parity.py::test_sharded_groups_compact_plus_unpermute.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_05016_b200.sharded import ShardPlan, gather_rows


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_plan_ranges_match_reference_split():
    # src/spmm.cpp:137-142: g_begin = G*w/workers
    for G in (1, 5, 32, 33, 256):
        for W in (1, 2, 3, 4, 8):
            plan = ShardPlan(G, 64, W)
            spans = [plan.range(r) for r in range(W)]
            assert spans[0][0] == 0 and spans[-1][1] == G
            assert all(spans[i][1] == spans[i + 1][0] for i in range(W - 1))
            assert all(b - a <= plan.chunk_groups for a, b in spans)


def test_row_map_marks_padding():
    plan = ShardPlan(5, 2, 2)  # ranks own 2 and 3 groups -> chunks of 3 groups
    ri = torch.arange(10, dtype=torch.int32).flip(0)
    m = plan.gathered_row_map(ri)
    assert m.shape[0] == 2 * 6
    assert m[:4].tolist() == ri[:4].tolist() and m[4:6].tolist() == [-1, -1]
    assert m[6:].tolist() == ri[4:].tolist()


def _worker(rank, world, port, M, K, N, V, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    from oracle import Oracle
    orc = Oracle()
    mask = orc.random_shflbw_mask(M, K, V, K // 4, orc.rng(1234))
    W = orc.round16(orc.random_dense(M, K, 1))
    B = orc.round16(orc.random_dense(K, N, 2))
    a = orc.compress(W, mask, V)
    plan = ShardPlan(M // V, V, world)
    g0, g1 = plan.range(rank)
    full_local = np.zeros((M, N), np.float32)
    orc.spmm_groups(a, B, g0, g1, full_local)  # this rank's worker share
    rows = a.row_indices[g0 * V: g1 * V].astype(np.int64)
    compact = torch.from_numpy(full_local[rows])  # group order
    gathered = gather_rows(plan, compact)
    row_map = plan.gathered_row_map(torch.from_numpy(a.row_indices.astype(np.int32)))
    out = torch.zeros((M, N))
    keep = row_map >= 0
    out[row_map[keep].long()] = gathered[keep]
    ok = np.array_equal(out.numpy(), orc.spmm(a, B))
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,M", [(2, 512), (3, 320)])
def test_gather_unpermute_gloo(world, M):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, 128, 24, 32, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, _ in res) == list(range(world))
    assert all(ok for _, ok in res)


def _fused_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2203_05016_b200 as sb
        from paper_2203_05016_b200.sharded import PeerOutputs, ShardedSpMM
        torch.cuda.set_device(0)
        g = torch.Generator().manual_seed(7)
        M, K, N, V = 1024, 512, 384, 64
        # the same synthetic layer on every rank: vector-wise groups, random columns
        mask = torch.zeros((M, K), dtype=torch.uint8)
        for grp in range(M // V):
            cols = torch.randperm(K, generator=g)[:K // 4]
            mask[grp * V:(grp + 1) * V, cols] = 1
        mask = mask[torch.randperm(M, generator=g)]
        W = (torch.rand((M, K), generator=g) * 2 - 1).to(torch.bfloat16).cuda()
        B = (torch.rand((K, N), generator=g) * 2 - 1).to(torch.bfloat16).cuda()
        a = sb.compress_shflbw(W, mask.cuda(), V)
        want = sb.spmm_execute(a, B, out_dtype=torch.bfloat16)
        outs = PeerOutputs((M, N), torch.bfloat16, world, rank)
        sh = ShardedSpMM(a, rank, world)
        got = sh.full_fused(B, outs)
        ok = bool(torch.equal(got, want))
        # a reader of the first result enqueued, then a second layer call that
        # overwrites every rank's buffer: the reader must see the first result
        snap = got.float() * 1.0
        B2 = (torch.rand((K, N), generator=g) * 2 - 1).to(torch.bfloat16).cuda()
        want2 = sb.spmm_execute(a, B2, out_dtype=torch.bfloat16)
        got2 = sh.full_fused(B2, outs)
        ok = ok and bool(torch.equal(snap, want.float())) and bool(torch.equal(got2, want2))
        q.put((rank, ok))
        dist.barrier()
        outs.close()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, f"error: {e!r}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_fused_allgather_two_processes_one_gpu():
    """The fused all-gather across processes: CUDA IPC handles exchanged over
    the process group, each rank's epilogue storing its rows into both
    ranks' full buffers.  Both ranks share cuda:0 here (the kernels never wait
    on each other; only the host barriers synchronise the ranks), so the
    IPC + P2P-pointer plumbing runs end to end on one GPU."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    world, port = 2, free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_fused_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


def _multicast_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    try:
        import paper_2203_05016_b200 as sb
        from paper_2203_05016_b200.sharded import MulticastOutputs, ShardedSpMM
        g = torch.Generator().manual_seed(9)
        M, K, N, V = 1024, 512, 384, 64
        mask = torch.zeros((M, K), dtype=torch.uint8)
        for grp in range(M // V):
            mask[grp * V:(grp + 1) * V, torch.randperm(K, generator=g)[:K // 4]] = 1
        mask = mask[torch.randperm(M, generator=g)]
        W = (torch.rand((M, K), generator=g) * 2 - 1).to(torch.bfloat16).cuda()
        B = (torch.rand((K, N), generator=g) * 2 - 1).to(torch.bfloat16).cuda()
        a = sb.compress_shflbw(W, mask.cuda(), V)
        want = sb.spmm_execute(a, B, out_dtype=torch.bfloat16)
        try:
            outs = MulticastOutputs((M, N), torch.bfloat16)
        except Exception as e:  # symmetric memory / multicast unavailable here
            q.put((rank, f"skip: {e!r}"))
            return
        if not outs.mc_ptr:
            q.put((rank, "skip: no multicast address (multicast_ptr == 0)"))
            return
        sh = ShardedSpMM(a, rank, world)
        got = sh.full_multicast(B, outs)
        ok = bool(torch.equal(got, want))
        got2 = sh.full_multicast(B, outs)  # again into the same buffers
        q.put((rank, ok and bool(torch.equal(got2, want)) and sb.last_plan().startswith("k_spmm")))
    except Exception as e:
        q.put((rank, f"error: {e!r}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_multicast_allgather_one_rank():
    """The NVLS multicast epilogue (multimem.st through torch symmetric
    memory's multicast address) with one rank: every row lands in the
    rank's own buffer exactly as spmm_execute writes it.  Skipped when the
    box offers no multicast object."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_multicast_worker, args=(0, 1, free_port(), q))
    p.start()
    rank, res = q.get(timeout=240)
    p.join(timeout=60)
    if isinstance(res, str) and res.startswith("skip"):
        pytest.skip(res)
    assert res is True, res
