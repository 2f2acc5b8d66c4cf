"""Multi-rank merge and sort at the BASELINE sizes, on the one-GPU lease.

The multi-GPU path (P2PMerger / P2PSorter: one process per GPU, peers'
shards mapped through CUDA IPC and read by the merge kernels themselves) is
run here with P processes sharing the box's one B200: every peer mapping is
a same-device IPC mapping, the kernels and the host protocol are the ones an
8xB200 node runs.  No kernel waits on another (host barriers order the
phases), so time-slicing the ranks on one GPU is safe.

  * config 5 (f32, |A| = |B| = 2^31, A ~ Normal, B ~ Exp, IEEE totalOrder)
    as 8 ranks, each holding 1/8 of A and of B and producing its 2^29-element
    slice of S; the concatenated slices are compared byte for byte with the
    REFERENCE's parallel_merge_into (oracle/_ref, totalOrder comparator,
    parallel.hpp:151-162) on the same input bytes.
  * config 4 (2^30 u32, seed 4) through P2PSorter at P = 2, 4, 8 (local
    sort of a 1/P shard + log2 P cross-rank Merge Path rounds,
    sort.hpp:132-148); the concatenated slices equal, byte for byte, the
    reference's own parallel_merge_sort of the keys (oracle/_ref).
  * config 3a (u64 keys + u32 values, 2^29 + 2^25) as 8 ranks: keys and
    values byte-compared with the reference's {key, value} merge.
  * all with the default loader choice (a rank's own shards through the
    bulk-copy engine, mapped peer shards through LSU loads) and with
    MP_PEER_LSU=1 (the LSU loader for every window).

The parent process owns the inputs and the output on cuda:0 and hands them
to the ranks as CUDA tensors (torch.multiprocessing shares them through
CUDA IPC); each rank copies its shard into its own allocation (exported to
its peers by the library) and writes its output slice back into the shared
output tensor.
"""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _release_parent_memory():
    """The parent holds up to ~100 GiB per test (inputs, output, oracle
    sorts): hand it back before the next test spawns its ranks."""
    yield
    import gc
    import torch
    from paper_1406_2628_b200 import _native as N
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    N.check(N.lib.mp_release(0))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_env(rank, world, port, peer_lsu):
    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if peer_lsu:
        os.environ["MP_PEER_LSU"] = "1"  # read once per process by the library
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return torch, dist


def _merge_rank(rank, world, port, peer_lsu, a_all, b_all, out_all, q):
    try:
        torch, dist = _rank_env(rank, world, port, peer_lsu)
        from paper_1406_2628_b200 import _native as N
        from paper_1406_2628_b200 import multigpu as mg
        na, nb = a_all.numel(), b_all.numel()
        a = a_all[rank * na // world:(rank + 1) * na // world].clone()
        b = b_all[rank * nb // world:(rank + 1) * nb // world].clone()
        torch.cuda.synchronize()
        m = mg.P2PMerger(a, b, key_type=N.KEY_F32)
        out, _ = m()
        assert out.numel() == m.o1 - m.o0
        out_all[m.o0:m.o1].copy_(out)
        torch.cuda.synchronize()
        m.close()
        dist.barrier()
        q.put((rank, "ok", (m.o0, m.o1)))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, "ERR", traceback.format_exc()))


def _merge_vals_rank(rank, world, port, peer_lsu, a_all, b_all, av_all, bv_all, out_all,
                     outv_all, q):
    try:
        torch, dist = _rank_env(rank, world, port, peer_lsu)
        from paper_1406_2628_b200 import _native as N
        from paper_1406_2628_b200 import multigpu as mg
        na, nb = a_all.numel(), b_all.numel()
        sa = slice(rank * na // world, (rank + 1) * na // world)
        sb = slice(rank * nb // world, (rank + 1) * nb // world)
        a, av = a_all[sa].clone(), av_all[sa].clone()
        b, bv = b_all[sb].clone(), bv_all[sb].clone()
        torch.cuda.synchronize()
        m = mg.P2PMerger(a, b, av, bv, key_type=N.KEY_U64)
        out, outv = m()
        out_all[m.o0:m.o1].copy_(out)
        outv_all[m.o0:m.o1].copy_(outv)
        torch.cuda.synchronize()
        m.close()
        dist.barrier()
        q.put((rank, "ok", (m.o0, m.o1)))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, "ERR", traceback.format_exc()))


def _sort_rank(rank, world, port, peer_lsu, x_all, out_all, q):
    try:
        torch, dist = _rank_env(rank, world, port, peer_lsu)
        from paper_1406_2628_b200 import _native as N
        from paper_1406_2628_b200 import multigpu as mg
        n = x_all.numel()
        lo, hi = rank * n // world, (rank + 1) * n // world
        x = x_all[lo:hi].clone()
        torch.cuda.synchronize()
        s = mg.P2PSorter((n + world - 1) // world + 1, torch.uint32, N.KEY_U32)
        out = s.run(x)
        lens = s.comm.all_gather_int([out.numel()])
        o0 = sum(v[0] for v in lens[:rank])
        out_all[o0:o0 + out.numel()].copy_(out)
        torch.cuda.synchronize()
        s.close()
        dist.barrier()
        q.put((rank, "ok", (o0, o0 + out.numel())))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, "ERR", traceback.format_exc()))


def _run_ranks(target, world, *args):
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port) + args + (q,))
             for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    try:
        for _ in range(world):
            r, status, info = q.get(timeout=900)
            assert status != "ERR", info
            got[r] = info
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():  # pragma: no cover
                p.kill()
    # the slices tile the output in rank order
    edges = [got[r] for r in range(world)]
    assert edges[0][0] == 0 and all(edges[r][1] == edges[r + 1][0] for r in range(world - 1))
    return edges


_REF_SORT = {}


def _reference_sort(keys):
    """oracle/_ref's parallel_merge_sort on this host's cores (cached: the
    six sorter tests share the config-4 keys); torch.sort where the
    reference library is not built."""
    if "c4" not in _REF_SORT:
        from oracle import bindings as B
        if B.REF_LIB.exists():
            _REF_SORT["c4"], _ = B.ref().merge_sort("u32", keys, p=B.host_cores())
        else:
            _REF_SORT["c4"] = np.sort(keys)
    return _REF_SORT["c4"]


def _gen_sorted_f32(kind, seed, n, dev):
    import torch
    from paper_1406_2628_b200 import _native as N
    st = torch.cuda.current_stream().cuda_stream
    x = torch.empty(n, dtype=torch.float32, device=dev)
    N.check(N.lib.mp_generate(kind, seed, 0, n, x.data_ptr(), st))
    N.check(N.lib.mp_sort(N.KEY_F32, x.data_ptr(), None, n, None, 0, st))
    return x


@pytest.mark.parametrize("peer_lsu", [False, True], ids=["default", "peer_lsu"])
def test_config5_eight_ranks_vs_reference(cuda, peer_lsu):
    import torch
    from oracle import bindings as B
    if not B.REF_LIB.exists():
        pytest.skip("oracle/_ref (the reference library) not built")
    n = 1 << 31
    a = _gen_sorted_f32(5, 1, n, cuda)   # A ~ Normal(0, 1), seed 1
    b = _gen_sorted_f32(6, 2, n, cuda)   # B ~ Exp(1), seed 2
    out = torch.full((2 * n,), float("nan"), dtype=torch.float32, device=cuda)
    torch.cuda.synchronize()
    edges = _run_ranks(_merge_rank, 8, peer_lsu, a, b, out)
    assert edges[-1][1] == 2 * n and all(e1 - e0 == n // 4 for e0, e1 in edges)
    ha, hb = a.cpu().numpy(), b.cpu().numpy()
    del a, b
    got = out.cpu().numpy()
    del out
    torch.cuda.empty_cache()
    R = B.ref()
    team = R.team(B.host_cores())
    want, _, _ = R.merge("f32", ha, hb, team=team)
    team.close()
    del ha, hb
    assert got.view(np.uint32).tobytes() == want.view(np.uint32).tobytes()


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("peer_lsu", [False, True], ids=["default", "peer_lsu"])
def test_config4_sorter_ranks(cuda, world, peer_lsu):
    import torch
    from paper_1406_2628_b200 import _native as N
    n = 1 << 30
    x = torch.empty(n, dtype=torch.uint32, device=cuda)
    N.check(N.lib.mp_generate(0, 4, 0, n, x.data_ptr(), torch.cuda.current_stream().cuda_stream))
    out = torch.zeros(n, dtype=torch.uint32, device=cuda)
    torch.cuda.synchronize()
    edges = _run_ranks(_sort_rank, world, peer_lsu, x, out)
    assert edges[-1][1] == n
    # the REFERENCE's parallel_merge_sort (sort.hpp:132-148) on the same
    # keys, computed once per session
    want = _reference_sort(x.cpu().numpy())
    del x
    assert out.cpu().numpy().tobytes() == want.tobytes()


def test_config3a_values_eight_ranks_vs_reference(cuda):
    """Config 3a (u64 keys + u32 values = source index, bit 31 marks B;
    |A| = 2^29, |B| = 2^25) as 8 ranks: keys and values byte-compared with
    the reference's parallel_merge_into on {key, value} records (stability
    across rank boundaries is visible in the values)."""
    import torch
    from oracle import bindings as B
    from paper_1406_2628_b200 import _native as N
    if not B.REF_LIB.exists():
        pytest.skip("oracle/_ref (the reference library) not built")
    st = torch.cuda.current_stream().cuda_stream
    na, nb = 1 << 29, 1 << 25

    def gen(seed, n):
        x = torch.empty(n, dtype=torch.uint64, device=cuda)
        N.check(N.lib.mp_generate(2, seed, 0, n, x.data_ptr(), st))
        N.check(N.lib.mp_sort(N.KEY_U64, x.data_ptr(), None, n, None, 0, st))
        return x

    a, b = gen(1, na), gen(2, nb)
    av = torch.arange(na, dtype=torch.int32, device=cuda).view(torch.uint32)
    bv = (torch.arange(nb, dtype=torch.int32, device=cuda)
          + torch.iinfo(torch.int32).min).view(torch.uint32)
    out = torch.zeros(na + nb, dtype=torch.uint64, device=cuda)
    outv = torch.zeros(na + nb, dtype=torch.uint32, device=cuda)
    torch.cuda.synchronize()
    _run_ranks(_merge_vals_rank, 8, False, a, b, av, bv, out, outv)
    ra = np.zeros(na, dtype=B.KV_DTYPE)
    ra["key"], ra["val"] = a.cpu().numpy(), av.cpu().numpy()
    rb = np.zeros(nb, dtype=B.KV_DTYPE)
    rb["key"], rb["val"] = b.cpu().numpy(), bv.cpu().numpy()
    del a, b, av, bv
    got, gotv = out.cpu().numpy(), outv.cpu().numpy()
    del out, outv
    team = B.ref().team(B.host_cores())
    want, _, _ = B.ref().merge("kv", ra, rb, team=team)
    team.close()
    assert np.array_equal(got, want["key"]) and np.array_equal(gotv, want["val"])
