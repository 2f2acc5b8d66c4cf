"""Multi-GPU Merge Path: one process per GPU over torch.distributed.

Theorem 14 / Corollary 6 of the paper applied at
GPU granularity: the merged output S is cut into P equal slices on the
cross diagonals d_r = floor(r*N/P); rank r finds its split (a_r, b_r) on
d_r, pulls A[a_r, a_{r+1}) and B[b_r, b_{r+1}) from whichever ranks own
them, and merges them locally with the single-GPU kernels.  Writes are
disjoint, so there is exactly ONE exchange per merge and no other
communication.

The three steps map onto the B200 box as:

  1. split search   -- all P-1 interior diagonals are searched jointly with a
                       K-ary search: per step every rank knows every probe
                       position (the state is replicated), fills the probe
                       keys it owns from its local shard (a device gather)
                       and one all_reduce(SUM) delivers them all.  A 2^31
                       diagonal needs ceil(31 / log2 K) steps (K = 64: 6).
  2. exchange       -- the split points give every (owner, receiver) slice;
                       one all_to_all_single per array (keys, then values)
                       moves them: NCCL grouped send/recv over NVLink 5 /
                       NVSwitch on the GPU box, gloo in the CPU tests.
  3. local merge    -- mp_merge on the received contiguous A and B ranges.

Sorting (config 4 at P GPUs): each rank sorts its shard with mp_sort, then
ceil(log2 P) rounds merge pairs of sorted rank-blocks with the same
sharded merge (left block = A, so the sort stays stable w.r.t. input order;
an unpaired last block is carried, as in sort.hpp:98-100).

The host logic here is backend-agnostic; the GPU-side work is the
library's kernels.  `local_merge` / `local_sort` hooks exist so the CPU
test-suite can run the distributed host logic over gloo with a checker in
place of the device kernels.
"""
from __future__ import annotations

import bisect
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native as N

K_ARY = 64  # probes per search step = K_ARY - 1


# --------------------------------------------------------------------------
# keys: order-preserving int64 image (so torch int64 compares implement the
# library's comparator: unsigned, signed, IEEE totalOrder, element key)
# --------------------------------------------------------------------------
def key_type_of(t: torch.Tensor, key_type=None) -> int:
    if key_type is not None:
        return key_type
    m = {torch.uint32: N.KEY_U32, torch.int32: N.KEY_I32, torch.float32: N.KEY_F32,
         torch.uint64: N.KEY_U64, torch.int64: N.KEY_I64}
    if t.dtype not in m:
        raise TypeError(f"unsupported key dtype {t.dtype}")
    return m[t.dtype]


def _flat_keys(t: torch.Tensor, kt: int) -> torch.Tensor:
    """Raw key words as a signed integer tensor of one element per key."""
    if kt in (N.KEY_U32, N.KEY_I32, N.KEY_F32):
        return t.view(torch.int32)
    if kt in (N.KEY_U64, N.KEY_I64):
        return t.view(torch.int64)
    return t.view(torch.int64).view(-1, 2)[:, 0]  # element: int64 key first


def order_image(raw: torch.Tensor, kt: int) -> torch.Tensor:
    """int64 image whose signed order equals the key order of `kt`."""
    x = raw.to(torch.int64)
    if kt == N.KEY_U32:
        return x & 0xFFFFFFFF
    if kt == N.KEY_I32:
        return x
    if kt == N.KEY_F32:
        u = x & 0xFFFFFFFF
        return torch.where((u & 0x80000000) != 0, u ^ 0xFFFFFFFF, u | 0x80000000)
    if kt == N.KEY_U64:
        return x ^ torch.iinfo(torch.int64).min
    return x  # I64, ELEMENT key


def n_keys(t: torch.Tensor, kt: int) -> int:
    return t.numel() * t.element_size() // N.KEY_SIZES[kt]


# --------------------------------------------------------------------------
# jobs: a merge of two sequences, each spread over an ordered list of ranks
# --------------------------------------------------------------------------
@dataclass
class Piece:
    rank: int
    start: int   # global index of this piece's first element in its sequence
    length: int


@dataclass
class Job:
    a: list          # [Piece] in sequence order (ascending rank)
    b: list          # [Piece]
    owners: list     # output ranks in order; slice k = [floor(k*N/m), floor((k+1)*N/m))

    @property
    def na(self) -> int:
        return sum(p.length for p in self.a)

    @property
    def nb(self) -> int:
        return sum(p.length for p in self.b)

    def diagonal(self, k: int) -> int:
        n = self.na + self.nb
        return k * n // len(self.owners)


def _pieces(ranks, lengths):
    out, s = [], 0
    for r in ranks:
        out.append(Piece(r, s, int(lengths[r])))
        s += int(lengths[r])
    return out


def _owner(pieces, idx):
    starts = [p.start for p in pieces]
    k = bisect.bisect_right(starts, idx) - 1
    while pieces[k].length == 0 or idx >= pieces[k].start + pieces[k].length:
        k += 1
    return pieces[k], idx - pieces[k].start


class _Comm:
    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        backend = dist.get_backend(group)
        self.dev = (torch.device("cuda", torch.cuda.current_device())
                    if backend == "nccl" else torch.device("cpu"))

    def all_gather_int(self, values):
        t = torch.tensor(values, dtype=torch.int64, device=self.dev)
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return [o.cpu().tolist() for o in out]

    def all_reduce_sum(self, t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def all_to_all(self, send: torch.Tensor, send_counts, recv_counts):
        # move raw words: signed integer views of the same width are supported
        # by every backend (gloo has no uint32/uint64 reductions or copies)
        wire = {1: torch.int8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[
            send.element_size()]
        recv = torch.empty(sum(recv_counts), dtype=wire, device=send.device)
        dist.all_to_all_single(recv, send.view(wire), recv_counts, send_counts,
                               group=self.group)
        return recv.view(send.dtype)


# --------------------------------------------------------------------------
# step 1: joint K-ary split search over all interior diagonals of all jobs
# --------------------------------------------------------------------------
def distributed_splits(comm: _Comm, jobs, a_local, b_local, kt, k_ary=K_ARY):
    """For each job, the a_off of the merge path on every owner boundary
    diagonal (k = 0..m).  Same predicate as the device kernels: move right
    iff B[d-1-m] < A[m] (ties to A, core.hpp:107-114)."""
    a_img_src = _flat_keys(a_local, kt) if a_local is not None else None
    b_img_src = _flat_keys(b_local, kt) if b_local is not None else None
    # search state: (job, k, d, lo, hi)
    searches = []
    result = []
    for j, job in enumerate(jobs):
        m = len(job.owners)
        res = [0] * (m + 1)
        res[m] = job.na
        for k in range(1, m):
            d = job.diagonal(k)
            lo, hi = max(0, d - job.nb), min(d, job.na)
            searches.append([j, k, d, lo, hi])
        result.append(res)
    while True:
        active = [s for s in searches if s[3] < s[4]]
        if not active:
            break
        # probe table: for every active search, its probe positions
        table = []  # (search, m)
        for s in active:
            lo, hi = s[3], s[4]
            span = hi - lo
            if span <= k_ary - 1:
                ms = list(range(lo, hi))
            else:
                ms = sorted(set(lo + (i * span) // k_ary for i in range(1, k_ary)))
            for m_ in ms:
                table.append((s, m_))
        # fill the probe keys this rank owns: A[m] and B[d-1-m]
        a_idx, a_pos, b_idx, b_pos = [], [], [], []
        for t, (s, m_) in enumerate(table):
            job = jobs[s[0]]
            pa, off_a = _owner(job.a, m_)
            if pa.rank == comm.rank:
                a_idx.append(off_a)
                a_pos.append(t)
            pb, off_b = _owner(job.b, s[2] - 1 - m_)
            if pb.rank == comm.rank:
                b_idx.append(off_b)
                b_pos.append(t)
        vals = torch.zeros(2 * len(table), dtype=torch.int64, device=comm.dev)
        if a_idx:
            src = order_image(a_img_src[torch.tensor(a_idx, device=a_img_src.device)], kt)
            vals[torch.tensor(a_pos, device=comm.dev) * 2] = src.to(comm.dev)
        if b_idx:
            src = order_image(b_img_src[torch.tensor(b_idx, device=b_img_src.device)], kt)
            vals[torch.tensor(b_pos, device=comm.dev) * 2 + 1] = src.to(comm.dev)
        comm.all_reduce_sum(vals)
        v = vals.view(-1, 2).cpu()
        take_b = (v[:, 1] < v[:, 0]).tolist()
        # narrow every active search: first probe whose predicate is true
        t = 0
        for s in active:
            lo, hi = s[3], s[4]
            new_lo, new_hi = None, hi
            prev = lo - 1
            while t < len(table) and table[t][0] is s:
                m_ = table[t][1]
                if new_lo is None and take_b[t]:
                    new_lo, new_hi = prev + 1, m_
                prev = m_
                t += 1
            if new_lo is None:
                new_lo = prev + 1
            s[3], s[4] = new_lo, new_hi
    for s in searches:
        result[s[0]][s[1]] = s[3]
    return result


# --------------------------------------------------------------------------
# step 2: the exchange plan
# --------------------------------------------------------------------------
def _send_recv_counts(comm: _Comm, jobs, splits, which):
    """Counts of `which` ('a'/'b') elements each rank sends to / receives
    from every other rank, plus this rank's local offsets to send."""
    P = comm.world
    send = [0] * P
    recv = [0] * P
    send_ranges = [None] * P  # local [lo, hi) sent to each receiver
    for job, spl in zip(jobs, splits):
        pieces = job.a if which == "a" else job.b
        for k, owner in enumerate(job.owners):
            if which == "a":
                lo, hi = spl[k], spl[k + 1]
            else:
                lo, hi = job.diagonal(k) - spl[k], job.diagonal(k + 1) - spl[k + 1]
            for pc in pieces:
                s = max(lo, pc.start)
                e = min(hi, pc.start + pc.length)
                if e <= s:
                    continue
                if pc.rank == comm.rank:
                    send[owner] += e - s
                    send_ranges[owner] = (s - pc.start, e - pc.start)
                if owner == comm.rank:
                    recv[pc.rank] += e - s
    return send, recv, send_ranges


def _gather_send(local, ranges, P, elem_view):
    parts = []
    for r in range(P):
        if ranges[r] is not None:
            lo, hi = ranges[r]
            parts.append(elem_view(local)[lo:hi])
    if not parts:
        return elem_view(local)[:0]
    return torch.cat(parts)


def _elem_view(kt):
    if kt == N.KEY_ELEMENT:
        return lambda t: t.view(torch.int64).view(-1, 2)
    return lambda t: t


# --------------------------------------------------------------------------
# step 3: local merge (device kernels by default)
# --------------------------------------------------------------------------
def _device_merge(a, b, av, bv, kt):
    from . import mergepath as mp
    if av is not None:
        return mp.parallel_merge(a, b, 1, a_vals=av, b_vals=bv, key_type=kt)
    return mp.parallel_merge(a, b, 1, key_type=kt), None


def _device_sort(x, v, kt):
    from . import mergepath as mp
    if v is not None:
        return mp.parallel_merge_sort(x, 1, vals=v, key_type=kt)
    return mp.parallel_merge_sort(x, 1, key_type=kt), None


def run_jobs(comm: _Comm, jobs, a_local, b_local, kt, a_vals=None, b_vals=None,
             local_merge=None):
    """Execute merge jobs; returns this rank's (keys, values) output slice."""
    splits = distributed_splits(comm, jobs, a_local, b_local, kt)
    ev = _elem_view(kt)
    outs_k, outs_v = [], []
    sa, ra, rng_a = _send_recv_counts(comm, jobs, splits, "a")
    sb, rb, rng_b = _send_recv_counts(comm, jobs, splits, "b")
    P = comm.world
    dev = comm.dev

    def xfer(local, send_c, recv_c, rngs, view):
        if local is None:
            local = torch.empty(0, dtype=torch.int32, device=dev)
        send = _gather_send(local, rngs, P, view).contiguous().to(dev)
        sc = send_c
        if view is not None and send.dim() == 2:
            flat = send.reshape(-1)
            got = comm.all_to_all(flat, [c * 2 for c in sc], [c * 2 for c in recv_c])
            return got.view(-1, 2)
        return comm.all_to_all(send, sc, recv_c)

    got_a = xfer(a_local, sa, ra, rng_a, ev)
    got_b = xfer(b_local, sb, rb, rng_b, ev)
    got_av = got_bv = None
    if a_vals is not None:
        got_av = xfer(a_vals, sa, ra, rng_a, lambda t: t)
        got_bv = xfer(b_vals, sb, rb, rng_b, lambda t: t)
    if kt == N.KEY_ELEMENT:
        got_a = got_a.reshape(-1)
        got_b = got_b.reshape(-1)
    if local_merge is None:
        # exchange buffers live on the backend's device (CPU for gloo);
        # the local merge runs where the shards live
        home = next((t.device for t in (a_local, b_local) if t is not None and t.is_cuda),
                    None)
        if home is not None:
            got_a, got_b = got_a.to(home), got_b.to(home)
            if got_av is not None:
                got_av, got_bv = got_av.to(home), got_bv.to(home)
    merge = local_merge or _device_merge
    k, v = merge(got_a, got_b, got_av, got_bv, kt)
    outs_k.append(k)
    outs_v.append(v)
    return outs_k[0], outs_v[0]


# --------------------------------------------------------------------------
# fused transport: peer-mapped shards read directly by the merge kernels
# --------------------------------------------------------------------------
def _export(t: torch.Tensor):
    import ctypes as C
    if t.numel() == 0:
        return None
    h = (C.c_char * 64)()
    off = C.c_uint64(0)
    N.check(N.lib.mp_ipc_export(t.data_ptr(), h, C.byref(off)))
    return bytes(h), off.value


def _import(rec) -> int:
    import ctypes as C
    if rec is None:
        return 0
    handle, off = rec
    p = C.c_void_p()
    buf = C.create_string_buffer(handle, 64)
    N.check(N.lib.mp_ipc_import(buf, off, C.byref(p)))
    return p.value or 0


class P2PMerger:
    """Multi-GPU merge with the exchange fused into the merge kernels.

    Every rank exports its A and B shards (CUDA IPC); every rank maps all
    peers' shards once (peer access over NVLink 5 / NVSwitch) and runs
    mp_merge_pieces on its output slice S[floor(rN/P), floor((r+1)N/P)):
    the piece-crossing probe reads peer keys directly and the K1/K2 tile
    loads pull their windows from peer HBM -- no all_to_all, no staging
    buffer, one kernel set per rank.  Barriers bracket each merge (inputs
    complete before anyone reads them; nobody reuses a shard while a peer
    may still read it)."""

    def __init__(self, a_local, b_local, a_vals=None, b_vals=None, key_type=None,
                 group=None):
        self.comm = _Comm(group)
        self.kt = key_type_of(a_local, key_type)
        self.a, self.b, self.av, self.bv = a_local, b_local, a_vals, b_vals
        me = (n_keys(a_local, self.kt), n_keys(b_local, self.kt), _export(a_local),
              _export(b_local), _export(a_vals) if a_vals is not None else None,
              _export(b_vals) if b_vals is not None else None)
        recs = [None] * self.comm.world
        dist.all_gather_object(recs, me, group=group)
        self.pa, self.pb = [], []
        for r, (la, lb, ea, eb, eav, ebv) in enumerate(recs):
            if r == self.comm.rank:
                ka, kb = a_local.data_ptr() if la else 0, b_local.data_ptr() if lb else 0
                va = a_vals.data_ptr() if a_vals is not None and la else None
                vb = b_vals.data_ptr() if b_vals is not None and lb else None
            else:
                ka, kb = _import(ea), _import(eb)
                va = _import(eav) if eav is not None else None
                vb = _import(ebv) if ebv is not None else None
            self.pa.append((ka or None, va, la))
            self.pb.append((kb or None, vb, lb))
        self.na = sum(p[2] for p in self.pa)
        self.nb = sum(p[2] for p in self.pb)
        n, P, r = self.na + self.nb, self.comm.world, self.comm.rank
        self.o0, self.o1 = r * n // P, (r + 1) * n // P
        self._arr_a = N.pieces_array(self.pa)
        self._arr_b = N.pieces_array(self.pb)

    def __call__(self, out=None, out_vals=None, sync=True):
        m = self.o1 - self.o0
        if out is None:
            out = torch.empty(m * (2 if self.kt == N.KEY_ELEMENT else 1),
                              dtype=self.a.dtype if self.kt != N.KEY_ELEMENT else torch.int64,
                              device=self.a.device)
        if out_vals is None and self.av is not None:
            out_vals = torch.empty(m, dtype=torch.uint32, device=self.a.device)
        stream = torch.cuda.current_stream(self.a.device)
        if sync:
            stream.synchronize()
            dist.barrier(group=self.comm.group)
        N.check(N.lib.mp_merge_pieces(self.kt, self._arr_a, len(self.pa), self._arr_b,
                                      len(self.pb), self.o0, self.o1, out.data_ptr(),
                                      out_vals.data_ptr() if out_vals is not None else None,
                                      stream.cuda_stream))
        if sync:
            stream.synchronize()
            dist.barrier(group=self.comm.group)
        return out, out_vals


class P2PSorter:
    """Multi-GPU stable merge sort with the exchange fused into the merges.

    Each rank owns two device buffers (ping/pong) of `capacity` keys, mapped
    into every peer once (CUDA IPC).  run(): local mp_sort of the rank's
    shard into ping, then ceil(log2 P) rounds; in round r, rank blocks of
    h = 2^r ranks are paired (left block = A, so the sort stays stable w.r.t.
    input order; an unpaired last block is carried, sort.hpp:98-100) and
    every rank of a pair merges its equal slice of the pair's output with
    mp_merge_pieces straight from the peers' mapped buffers into its pong
    buffer.  A barrier closes each round (nobody overwrites a buffer a peer
    may still read), then ping/pong swap.  Slice sizes are computed, not
    communicated: every rank knows every length."""

    def __init__(self, capacity: int, dtype, key_type: int, group=None, device=None):
        self.comm = _Comm(group)
        self.kt = key_type
        self.capacity = int(capacity)
        dev = device or torch.device("cuda", torch.cuda.current_device())
        words = capacity * (2 if key_type == N.KEY_ELEMENT else 1)
        wdt = torch.int64 if key_type == N.KEY_ELEMENT else dtype
        self.buf = [torch.empty(max(words, 1), dtype=wdt, device=dev) for _ in range(2)]
        recs = [None] * self.comm.world
        dist.all_gather_object(recs, (_export(self.buf[0]), _export(self.buf[1])), group=group)
        self.peer = [[0, 0] for _ in range(self.comm.world)]
        for r, (e0, e1) in enumerate(recs):
            if r == self.comm.rank:
                self.peer[r] = [self.buf[0].data_ptr(), self.buf[1].data_ptr()]
            else:
                self.peer[r] = [_import(e0), _import(e1)]
        self.scratch = None

    def run(self, x_local: torch.Tensor, sync=True):
        P, me = self.comm.world, self.comm.rank
        kt = self.kt
        n_me = n_keys(x_local, kt)
        if n_me > self.capacity:
            # buf[0] holds `capacity` keys and is mapped into every peer:
            # an overrun would corrupt memory the peers read
            raise ValueError(f"P2PSorter.run: shard of {n_me} keys exceeds the capacity "
                             f"{self.capacity} set at construction")
        lens = [x[0] for x in self.comm.all_gather_int([n_me])]
        stream = torch.cuda.current_stream(self.buf[0].device)
        st = stream.cuda_stream
        sb = N.lib.mp_sort_scratch_bytes(kt, 0, n_me)
        if self.scratch is None or self.scratch.numel() < max(sb, 16):
            self.scratch = torch.empty(max(sb, 16), dtype=torch.uint8, device=self.buf[0].device)
        N.check(N.lib.mp_sort_to(kt, x_local.data_ptr(), None, self.buf[0].data_ptr(), None,
                                 n_me, self.scratch.data_ptr(), self.scratch.numel(), st))
        cur, h = 0, 1
        while h < P:
            if sync:
                stream.synchronize()
                dist.barrier(group=self.comm.group)
            new_lens = list(lens)
            s0 = (me // (2 * h)) * 2 * h
            left = list(range(s0, min(s0 + h, P)))
            right = list(range(s0 + h, min(s0 + 2 * h, P)))
            for s in range(0, P, 2 * h):  # every block pair's new slice sizes
                L = list(range(s, min(s + h, P)))
                R = list(range(s + h, min(s + 2 * h, P)))
                if R:
                    owners = L + R
                    tot = sum(lens[q] for q in owners)
                    for k, q in enumerate(owners):
                        new_lens[q] = (k + 1) * tot // len(owners) - k * tot // len(owners)
            if right:
                owners = left + right
                k = owners.index(me)
                tot = sum(lens[q] for q in owners)
                o0, o1 = k * tot // len(owners), (k + 1) * tot // len(owners)
                if o1 - o0 > self.capacity:  # an equal split never exceeds the largest shard
                    raise ValueError("P2PSorter.run: round slice exceeds the capacity")
                pa = N.pieces_array([(self.peer[q][cur] if lens[q] else None, None, lens[q])
                                     for q in left])
                pb = N.pieces_array([(self.peer[q][cur] if lens[q] else None, None, lens[q])
                                     for q in right])
                N.check(N.lib.mp_merge_pieces(kt, pa, len(left), pb, len(right), o0, o1,
                                              self.buf[1 - cur].data_ptr(), None, st))
            else:  # carried block: copy through so every rank sits in `1-cur`
                words = lens[me] * (2 if kt == N.KEY_ELEMENT else 1)
                self.buf[1 - cur][:words].copy_(self.buf[cur][:words])
            lens = new_lens
            cur = 1 - cur
            h *= 2
        if sync:
            stream.synchronize()
            dist.barrier(group=self.comm.group)
        words = lens[me] * (2 if kt == N.KEY_ELEMENT else 1)
        return self.buf[cur][:words]


# --------------------------------------------------------------------------
# public API
# --------------------------------------------------------------------------
def sharded_merge(a_local: torch.Tensor, b_local: torch.Tensor, a_vals=None, b_vals=None,
                  key_type=None, group=None, local_merge=None, transport="nccl"):
    """Merge two sorted sequences sharded contiguously across the ranks
    (rank r holds A[offA_r, offA_r + |A_r|) and B likewise).  Rank r
    returns S[floor(r*N/P), floor((r+1)*N/P)) of the stable merge (ties: A
    first), plus the values that travel with the keys.

    transport="nccl": joint split search + all_to_all exchange + local merge
    (works on any backend, incl. gloo for the CPU tests).
    transport="p2p": shards mapped over NVLink (CUDA IPC) and pulled by the
    merge kernels themselves (P2PMerger); build the merger once to reuse
    the mappings across calls."""
    if transport == "p2p":
        return P2PMerger(a_local, b_local, a_vals, b_vals, key_type, group)()
    comm = _Comm(group)
    kt = key_type_of(a_local, key_type)
    lens = comm.all_gather_int([n_keys(a_local, kt), n_keys(b_local, kt)])
    ranks = list(range(comm.world))
    job = Job(_pieces(ranks, [x[0] for x in lens]), _pieces(ranks, [x[1] for x in lens]),
              ranks)
    return run_jobs(comm, [job], a_local, b_local, kt, a_vals, b_vals, local_merge)


def sharded_sort(x_local: torch.Tensor, vals=None, key_type=None, group=None,
                 local_sort=None, local_merge=None):
    """Stable sort of a sequence sharded contiguously across the ranks.
    Rank r ends with its slice of the globally sorted sequence (sizes of the
    final round's equal split).  Local sort, then ceil(log2 P) rounds of
    pairwise sharded merges of sorted rank-blocks (left block = A)."""
    comm = _Comm(group)
    kt = key_type_of(x_local, key_type)
    sort = local_sort or _device_sort
    keys, v = sort(x_local, vals, kt)
    P = comm.world
    h = 1
    while h < P:
        lens = comm.all_gather_int([n_keys(keys, kt)])
        lens = [x[0] for x in lens]
        jobs, mine = [], None
        for s in range(0, P, 2 * h):
            left = list(range(s, min(s + h, P)))
            right = list(range(s + h, min(s + 2 * h, P)))
            if not right:
                continue  # unpaired block carried (sort.hpp:98-100)
            job = Job(_pieces(left, lens), _pieces(right, lens), left + right)
            jobs.append(job)
            if comm.rank in left + right:
                mine = job
        in_left = mine is not None and comm.rank in [p.rank for p in mine.a]
        a_loc = keys if in_left else keys[:0]
        b_loc = keys if (mine is not None and not in_left) else keys[:0]
        av = bv = None
        if v is not None:
            av = v if in_left else v[:0]
            bv = v if (mine is not None and not in_left) else v[:0]
        if mine is None:
            # carried block still takes part in the collectives
            run_jobs(comm, jobs, keys[:0], keys[:0], kt,
                     v[:0] if v is not None else None, v[:0] if v is not None else None,
                     local_merge=lambda a, b, x, y, k: (a, x))
        else:
            keys, v = run_jobs(comm, jobs, a_loc, b_loc, kt, av, bv, local_merge)
        h *= 2
    return keys, v


# --------------------------------------------------------------------------
# bench.py --gpus N (N > 1): weak scaling, one process per GPU over NCCL
# --------------------------------------------------------------------------
class _NoClock:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False

    def summary(self):
        return None


def bench_distributed(args, cfg, ws, rank, local, clock=None):
    """Each rank holds a fixed-size shard (the config's |A| and |B| per GPU)
    of globally sorted A and B (generated with the SplitMix64 counter
    generator at the rank's global offsets, then sorted across the ranks
    with sharded_sort -- untimed).  A timed step is one sharded_merge: joint
    split search + NVLink exchange + local K1/K2 merge.  Max over ranks."""
    import json
    import statistics
    import time
    from pathlib import Path

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    kt = {"u32": N.KEY_U32, "i32": N.KEY_I32, "f32": N.KEY_F32, "u64": N.KEY_U64,
          "i64": N.KEY_I64}[cfg["key"]]
    dt = {"u32": torch.uint32, "i32": torch.int32, "f32": torch.float32,
          "u64": torch.uint64, "i64": torch.int64}[cfg["key"]]
    st = torch.cuda.current_stream().cuda_stream

    def gen(kind, seed, n, first):
        x = torch.empty(n, dtype=dt, device=dev)
        N.check(N.lib.mp_generate(kind, seed, first, n, x.data_ptr(), st))
        return x

    import os
    # MP_BENCH_SCALE=k shrinks the per-GPU sizes by 2^k (multi-rank smoke
    # tests on a one-GPU box); reductions go through the backend's device
    shrink = int(os.environ.get("MP_BENCH_SCALE", "0"))
    # config 5 fixes the global sizes (sharded over the ranks: strong
    # scaling); the others fix the per-GPU sizes (weak scaling)
    strong = bool(cfg.get("sharded"))
    NA, NB = cfg["na"] >> shrink, cfg["nb"] >> shrink
    if strong:
        a0, a1 = rank * NA // ws, (rank + 1) * NA // ws
        b0, b1 = rank * NB // ws, (rank + 1) * NB // ws
    else:
        a0, a1, b0, b1 = rank * NA, (rank + 1) * NA, rank * NB, (rank + 1) * NB
    na, nb = a1 - a0, b1 - b0
    red_dev = dev if dist.get_backend() == "nccl" else torch.device("cpu")
    a, _ = sharded_sort(gen(cfg["gen"][0], 1, na, a0), key_type=kt)
    b, _ = sharded_sort(gen(cfg["gen"][1], 2, nb, b0), key_type=kt)
    a, b = a.contiguous(), b.contiguous()
    av = bv = None
    if cfg.get("vals"):
        # config 3 payload: each key's index in its globally sorted array
        # (bit 31 set on B's), as in the single-GPU bench
        comm = _Comm()
        la = [x[0] for x in comm.all_gather_int([a.numel()])]
        lb = [x[0] for x in comm.all_gather_int([b.numel()])]
        av = (torch.arange(a.numel(), dtype=torch.int64, device=dev) + sum(la[:rank])
              ).to(torch.int32).view(torch.uint32)
        bv = ((torch.arange(b.numel(), dtype=torch.int64, device=dev) + sum(lb[:rank]))
              | (1 << 31)).to(torch.int32).view(torch.uint32)
    transport = getattr(args, "transport", "p2p")
    if transport == "p2p":
        merger = P2PMerger(a, b, av, bv, key_type=kt)  # IPC mappings built once (untimed)
        step = lambda: merger()  # noqa: E731
    else:
        step = lambda: sharded_merge(a, b, av, bv, key_type=kt)  # noqa: E731
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    times = []
    c0 = N.lib.mp_launch_count()
    with (clock or _NoClock)() as clk:
        for _ in range(args.steps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            out, _ = step()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    launches = N.lib.mp_launch_count() - c0
    dist.barrier()
    ms = torch.tensor([sum(times)], dtype=torch.float64, device=red_dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    total = (NA + NB) if strong else (na + nb) * ws
    value = total * args.steps / (ms / 1e3)
    # e2e through the public API with host buffers: H2D shard, sharded merge,
    # D2H of this rank's output slice (wall clock, max over ranks)
    ha, hb = a.cpu().pin_memory(), b.cpu().pin_memory()
    hav = av.cpu().pin_memory() if av is not None else None
    hbv = bv.cpu().pin_memory() if bv is not None else None
    e2e_steps = max(1, min(args.steps, getattr(args, "e2e_steps", 3)))
    dist.barrier()
    t = time.perf_counter()
    for _ in range(e2e_steps):
        a.copy_(ha, non_blocking=True)  # H2D into the registered shards
        b.copy_(hb, non_blocking=True)
        if hav is not None:
            av.copy_(hav, non_blocking=True)
            bv.copy_(hbv, non_blocking=True)
        o, ov = step()
        ho = o.cpu()
        if ov is not None:
            ho = ov.cpu()
    torch.cuda.synchronize()
    el = torch.tensor([time.perf_counter() - t], dtype=torch.float64, device=red_dev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    ks = a.element_size() + (4 if av is not None else 0)  # key (+ value) bytes
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json")
                      .read_text())["hbm_gbs"] if (Path(__file__).resolve().parents[1] /
                                                   "MEASURED_PEAKS.json").exists() else 6650.0
    per_rank_bytes = (na + nb) * 2 * ks
    achieved = per_rank_bytes / (ms / args.steps / 1e3) / 1e9
    del ho, statistics
    return {
        "metric": "merged elements/s", "value": value, "unit": "elements/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": cfg["key"],
        "data": "synthetic: SplitMix64 counter generator, globally sorted with sharded_sort",
        "config": {"workload": cfg["desc"] + (f"; sharded over {ws} GPUs" if strong else
                                             f" per GPU; global |A|={NA * ws} |B|={NB * ws}"),
                   "parallelism": f"merge-path diagonal split over {ws} GPUs ("
                                  + ("NVLink pull fused into the merge kernels via CUDA IPC"
                                     if transport == "p2p" else "NCCL all_to_all exchange") + ")",
                   "l2": "inputs+output larger than L2 (no flush needed)"},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm+nvlink", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "note": "per-rank algorithmic HBM bytes / step time; the exchange also "
                             "moves up to 4 B per remote element over NVLink"},
        "clocks": clk.summary(),
        "e2e": {"value": total * e2e_steps / float(el.item()), "unit": "elements/s",
                "h2d_bytes_per_step": (na + nb) * ks, "d2h_bytes_per_step": (na + nb) * ks},
    }


def bench_distributed_sort(args, cfg, ws, rank, local, clock=None):
    """bench.py --config 4 --gpus N: strong scaling of the 2^30-key sort
    (BASELINE config 4: each GPU local-sorts a 1/P shard, then Merge Path
    rounds across GPUs).  Shard r = keys [r*n/P, (r+1)*n/P) of the seed-4
    SplitMix64 sequence; a timed step = P2PSorter.run (local sort + log2 P
    fused NVLink merge rounds), max over ranks."""
    import os
    import time
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    shrink = int(os.environ.get("MP_BENCH_SCALE", "0"))
    n = cfg["n"] >> shrink
    lo, hi = rank * n // ws, (rank + 1) * n // ws
    x = torch.empty(hi - lo, dtype=torch.uint32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    N.check(N.lib.mp_generate(cfg["gen"][0], 4, lo, hi - lo, x.data_ptr(), st))
    sorter = P2PSorter((n + ws - 1) // ws + 1, torch.uint32, N.KEY_U32)
    for _ in range(args.warmup):
        sorter.run(x)
    torch.cuda.synchronize()
    dist.barrier()
    times = []
    c0 = N.lib.mp_launch_count()
    with (clock or _NoClock)() as clk:
        for _ in range(args.steps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            sorter.run(x)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    launches = N.lib.mp_launch_count() - c0
    red_dev = dev if dist.get_backend() == "nccl" else torch.device("cpu")
    ms = torch.tensor([sum(times)], dtype=torch.float64, device=red_dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    # e2e: pinned host shard -> device, sort, sorted slice back to the host
    hx = x.cpu().pin_memory()
    dist.barrier()
    t = time.perf_counter()
    e2e_steps = max(1, min(args.steps, getattr(args, "e2e_steps", 3)))
    for _ in range(e2e_steps):
        x.copy_(hx, non_blocking=True)
        o = sorter.run(x)
        ho = o.cpu()
    torch.cuda.synchronize()
    el = torch.tensor([time.perf_counter() - t], dtype=torch.float64, device=red_dev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    del ho
    rounds, w = 0, 8192  # mp_sort's bare 32-bit block-sort run
    while w < (n + ws - 1) // ws:
        w, rounds = 2 * w, rounds + 1
    passes = 1 + rounds + (ws - 1).bit_length()
    return {
        "metric": "merge-sort keys/s", "value": n * args.steps / (ms / 1e3), "unit": "keys/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32",
        "data": "synthetic: SplitMix64 counter generator, seed 4",
        "config": {"workload": cfg["desc"] + f"; {ws} GPUs, 1/{ws} shard each",
                   "parallelism": f"local sort + {(ws - 1).bit_length()} cross-GPU Merge Path "
                                  "rounds, NVLink pull fused into the merge (CUDA IPC)",
                   "l2": "inputs+output larger than L2 (no flush needed)"},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm+nvlink", "unit": "GB/s",
                     "achieved": (n // ws) * 8 * passes / (ms / args.steps / 1e3) / 1e9,
                     "peak": 6554.2, "frac": (n // ws) * 8 * passes / (ms / args.steps / 1e3)
                     / 1e9 / 6554.2, "traffic": None,
                     "note": f"per-GPU {passes} passes x 8 B/key over the step time"},
        "clocks": clk.summary(),
        "e2e": {"value": n * e2e_steps / float(el.item()), "unit": "keys/s",
                "h2d_bytes_per_step": (hi - lo) * 4, "d2h_bytes_per_step": (hi - lo) * 4},
    }
