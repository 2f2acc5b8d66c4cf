"""The fused multi-GPU merge path on the GPU box.

1. mp_merge_pieces in one process: A and B split into separately allocated
   pieces (what peer-mapped shards look like to the kernels) with ragged and
   empty pieces; every output range must equal the oracle's merge slice.
2. P2PMerger across two processes sharing the box's GPU: CUDA IPC maps each
   rank's shards into the other; each rank merges its output slice straight
   from the mapped pieces.  (One GPU is available to this run, so the peer
   mapping is same-device IPC; the kernels and the host protocol are the
   ones an 8xB200 node runs, with NVLink carrying the remote reads.  No
   kernel waits on another: host barriers order the phases.)
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


def _split_sizes(rng, n, k):
    cuts = np.sort(rng.integers(0, n + 1, k - 1))
    return np.diff(np.concatenate([[0], cuts, [n]])).tolist()


@pytest.mark.parametrize("kt_name", ["u32", "i32", "f32", "u64", "i64", "el"])
def test_merge_pieces_in_process(cuda, port, kt_name):
    import torch
    from paper_1406_2628_b200 import _native as N
    from test_gpu_parity import _rand_sorted, key_type, same, to_dev, from_dev
    rng = np.random.default_rng(41)
    kt = key_type(kt_name)
    st = torch.cuda.current_stream().cuda_stream
    # the last two: every tile straddles several (often empty) pieces
    for na, nb, npa, npb, dup in ((50_000, 37_001, 3, 5, 100), (200_001, 0, 4, 1, 7),
                                  (1 << 20, 1 << 19, 8, 8, 1 << 30), (5, 300_000, 2, 16, 3),
                                  (40, 33, 16, 16, 5), (3000, 2999, 16, 11, 1 << 20)):
        a = _rand_sorted(kt_name, rng, na, dup)
        b = _rand_sorted(kt_name, rng, nb, dup)
        if kt_name == "el":
            b["tag"] += np.uint32(1 << 24)
        want, _, _, _ = port.merge(kt_name, a, b)
        sa, sb = _split_sizes(rng, na, npa), _split_sizes(rng, nb, npb)
        keep = []

        def pieces(x, sizes):
            out, s = [], 0
            for ln in sizes:
                t = to_dev(x[s:s + ln], kt_name, cuda) if ln else None
                keep.append(t)
                out.append((t.data_ptr() if t is not None else None, None, ln))
                s += ln
            return N.pieces_array(out)

        pa, pb = pieces(a, sa), pieces(b, sb)
        n = na + nb
        for o0, o1 in ((0, n), (n // 3, 2 * n // 3), (n - 1, n), (7, 7)):
            m = o1 - o0
            out = to_dev(want[:max(m, 1)], kt_name, cuda).clone()
            N.check(N.lib.mp_merge_pieces(kt, pa, npa, pb, npb, o0, o1, out.data_ptr(), None, st))
            torch.cuda.synchronize()
            if m:
                assert same(from_dev(out, kt_name)[:m], want[o0:o1]), (kt_name, na, nb, o0, o1)


def test_merge_pieces_with_values(cuda, port):
    import torch
    from paper_1406_2628_b200 import _native as N
    rng = np.random.default_rng(43)
    st = torch.cuda.current_stream().cuda_stream
    na, nb = 300_000, 100_003
    a = np.sort(rng.integers(0, 50, na).astype(np.uint64))
    b = np.sort(rng.integers(0, 50, nb).astype(np.uint64))
    av = np.arange(na, dtype=np.uint32)
    bv = np.arange(nb, dtype=np.uint32) | np.uint32(1 << 31)
    want, wantv, _, _ = port.merge("u64", a, b, av=av, bv=bv)
    keep = []

    def pieces(x, v, sizes):
        out, s = [], 0
        for ln in sizes:
            tk = torch.from_numpy(x[s:s + ln].copy()).cuda()
            tv = torch.from_numpy(v[s:s + ln].copy()).cuda()
            keep.extend([tk, tv])
            out.append((tk.data_ptr() if ln else None, tv.data_ptr() if ln else None, ln))
            s += ln
        return N.pieces_array(out)

    for sa, sb in (([100_000, 0, 200_000], [1, 50_000, 50_002]),
                   ([1, 2, 3, 0, 5, 299_989], [7, 0, 0, 100_003 - 11, 1, 3])):
        pa, pb = pieces(a, av, sa), pieces(b, bv, sb)
        out = torch.empty(na + nb, dtype=torch.uint64, device=cuda)
        outv = torch.empty(na + nb, dtype=torch.uint32, device=cuda)
        N.check(N.lib.mp_merge_pieces(N.KEY_U64, pa, len(sa), pb, len(sb), 0, na + nb,
                                      out.data_ptr(), outv.data_ptr(), st))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), want)
        assert np.array_equal(outv.cpu().numpy(), wantv)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _p2p_worker(rank, world, port, q):
    try:
        sys.path.insert(0, str(ROOT))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1406_2628_b200 import _native as N
        from paper_1406_2628_b200 import multigpu as mg
        rng = np.random.default_rng(7)
        na, nb = 3_000_001, 2_000_000
        a = np.sort(rng.integers(0, 1 << 16, na).astype(np.int32))
        b = np.sort(rng.integers(0, 1 << 16, nb).astype(np.int32))
        ca = [0, 1_200_000, na]
        cb = [0, 1_700_000, nb]
        al = torch.from_numpy(a[ca[rank]:ca[rank + 1]].copy()).cuda()
        bl = torch.from_numpy(b[cb[rank]:cb[rank + 1]].copy()).cuda()
        av = torch.arange(ca[rank], ca[rank + 1], dtype=torch.int32).cuda().view(torch.uint32)
        bv = (torch.arange(cb[rank], cb[rank + 1], dtype=torch.int64) | (1 << 31)).to(
            torch.int64).numpy().astype(np.uint32)
        bv = torch.from_numpy(bv).cuda()
        m = mg.P2PMerger(al, bl, av, bv, key_type=N.KEY_I32)
        out, outv = m()
        out2, outv2 = m()  # reuse of the mappings
        assert torch.equal(out, out2) and torch.equal(outv, outv2)
        q.put((rank, out.cpu().numpy().tobytes(), outv.cpu().numpy().tobytes()))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, "ERR", traceback.format_exc()))


def test_p2p_merger_two_processes(cuda, port):
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, k, v = q.get(timeout=600)
        assert k != "ERR", v
        res[r] = (k, v)
    for p in procs:
        p.join(timeout=120)
    rng = np.random.default_rng(7)
    na, nb = 3_000_001, 2_000_000
    a = np.sort(rng.integers(0, 1 << 16, na).astype(np.int32))
    b = np.sort(rng.integers(0, 1 << 16, nb).astype(np.int32))
    want, wantv, _, _ = port.merge("i32", a, b, av=np.arange(na, dtype=np.uint32),
                                   bv=np.arange(nb, dtype=np.uint32) | np.uint32(1 << 31))
    got = np.frombuffer(res[0][0] + res[1][0], dtype=np.int32)
    gotv = np.frombuffer(res[0][1] + res[1][1], dtype=np.uint32)
    assert np.array_equal(got, want)
    assert np.array_equal(gotv, wantv)
    n = na + nb
    assert len(res[0][0]) // 4 == n // 2


def _sort_worker(rank, world, port, sizes, q):
    try:
        sys.path.insert(0, str(ROOT))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1406_2628_b200 import _native as N
        from paper_1406_2628_b200 import multigpu as mg
        rng = np.random.default_rng(11)
        x = rng.integers(0, 1 << 20, sum(sizes)).astype(np.uint32)
        cut = np.concatenate([[0], np.cumsum(sizes)])
        xl = torch.from_numpy(x[cut[rank]:cut[rank + 1]].copy()).cuda()
        s = mg.P2PSorter(max(sizes), torch.uint32, N.KEY_U32)
        out = s.run(xl)
        out2 = s.run(xl)  # buffers and mappings reused
        assert torch.equal(out, out2)
        q.put((rank, out.cpu().numpy().tobytes(), None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, "ERR", traceback.format_exc()))


@pytest.mark.parametrize("sizes", [[700_001, 699_999], [500_000, 20_000, 480_000],
                                   [300_000, 300_000, 300_000, 300_000]])
def test_p2p_sorter_processes(cuda, sizes):
    import torch.multiprocessing as tmp
    world = len(sizes)
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_sort_worker, args=(r, world, port_no, sizes, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, k, v = q.get(timeout=600)
        assert k != "ERR", v
        res[r] = k
    for p in procs:
        p.join(timeout=120)
    rng = np.random.default_rng(11)
    x = rng.integers(0, 1 << 20, sum(sizes)).astype(np.uint32)
    got = np.frombuffer(b"".join(res[r] for r in range(world)), dtype=np.uint32)
    assert np.array_equal(got, np.sort(x))


def test_signal_kernel_fallback_subprocess(cuda):
    """mp_signal's kernel fallback (a system-scope release store, used when
    the driver refuses a stream write to an address) forced on for the
    multi-process merger and sorter (MP_SIGNAL_KERNEL=1, read once per
    process)."""
    import subprocess
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", str(Path(__file__)),
                        "-k", "p2p_merger or p2p_sorter"], capture_output=True, text=True,
                       timeout=900, env=dict(os.environ, MP_SIGNAL_KERNEL="1"), cwd=str(ROOT))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def test_peer_lsu_loader_subprocess(cuda):
    """The peer-memory loader of K2 (LSU vector loads instead of bulk
    copies; chosen for windows on another GPU) forced on for every piece
    merge (MP_PEER_LSU=1, read once per process) on the in-process piece
    tests and the two-process P2P merger."""
    import subprocess
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", str(Path(__file__)),
                        "-k", "pieces or p2p_merger"], capture_output=True, text=True,
                       timeout=900, env=dict(os.environ, MP_PEER_LSU="1"), cwd=str(ROOT))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.parametrize("config", ["2", "3a", "4", "5"])
def test_distributed_bench_two_ranks(cuda, config):
    """bench.py --gpus 2 through torchrun (both ranks on the box's one GPU,
    gloo plumbing, inputs shrunk 2^5): the fused P2P merge (config 2, weak
    scaling; config 5, f32, the fixed global size sharded) and the P2P sort
    (config 4) run and print one JSON line with the library's launch count,
    the per-rank NVLink bytes from the actual split points and the
    HBM + NVLink roofline; config 2 also carries config 5 and the sort."""
    import json
    import subprocess
    env = dict(os.environ, MP_BENCH_DEVICE="0", MP_BENCH_BACKEND="gloo", MP_BENCH_SCALE="5")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(_free_port()), "bench.py", "--config", config, "--gpus", "2",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True,
                       timeout=900, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["scaling"] == ("weak" if config in ("2", "3a") else "strong")
    recs = [d] + ([d["config5"], d["sort"]] if config == "2" else [])
    for x in recs:
        rf = x["roofline"]
        assert rf["bound"] == "hbm+nvlink" and rf["nvlink_gbs"] > 0 and rf["peak"] > 0
        assert 0 < rf["frac"] and len(rf["t_g_ms"]) == 2
        assert len(x["nvlink"]["in_bytes_per_rank"]) == 2
    if config == "5":  # the ranks' output slices need the other rank's shards
        assert sum(d["nvlink"]["in_bytes_per_rank"]) > 0


def test_bench_gpus_flag_spawns_ranks(cuda):
    """`python bench.py --gpus 2` with no launcher starts its own two ranks
    (never silently runs one GPU); a WORLD_SIZE that disagrees is an error."""
    import json
    import subprocess
    env = dict(os.environ, MP_BENCH_DEVICE="0", MP_BENCH_BACKEND="gloo", MP_BENCH_SCALE="6")
    r = subprocess.run([sys.executable, "bench.py", "--config", "4", "--gpus", "2", "--steps",
                        "2", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                       env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["n_gpus"] == 2
    bad = subprocess.run([sys.executable, "bench.py", "--gpus", "4"], capture_output=True,
                         text=True, timeout=120, cwd=str(ROOT),
                         env=dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"))
    assert bad.returncode == 2
