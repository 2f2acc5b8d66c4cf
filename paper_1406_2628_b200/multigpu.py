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
from ctypes import c_void_p as C_void_p
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


class _Flags:
    """Stream-ordered phase barriers across ranks, with no host involvement.

    Every rank owns a device array of 2*P generation words (a READY and a
    DONE slot per peer), exported once through CUDA IPC and mapped by every
    peer.  arrive(phase, ranks) enqueues, on the caller's stream, one
    mp_signal per rank in `ranks` (a fenced write of the generation into
    that rank's slot for me) and one mp_wait per rank (the stream waits
    until my slot for that rank holds the generation).  All ranks call
    arrive() in the same sequence, so the generation -- a local counter --
    agrees across ranks; slots only grow, so a rank that runs ahead never
    confuses a slower one (waits are >=)."""

    READY, DONE = 0, 1

    def __init__(self, comm, device):
        self.comm = comm
        P = comm.world
        self.words = torch.zeros(2 * P, dtype=torch.int64, device=device)
        recs = [None] * P
        dist.all_gather_object(recs, _export(self.words), group=comm.group)
        self.base = [self.words.data_ptr() if r == comm.rank else _import(rec)
                     for r, rec in enumerate(recs)]
        self.imported = [b for r, b in enumerate(self.base) if r != comm.rank]
        self.gen = 0
        torch.cuda.synchronize(device)  # the zeroed words exist before any peer signals

    def slot(self, owner, phase, peer):
        return self.base[owner] + 8 * (phase * self.comm.world + peer)

    def arrive(self, phase, ranks, stream):
        self.gen += 1
        me = self.comm.rank
        for r in ranks:
            N.check(N.lib.mp_signal(self.slot(r, phase, me), self.gen, stream))
        for q in ranks:
            N.check(N.lib.mp_wait(self.slot(me, phase, q), self.gen, stream))


class P2PMerger:
    """Multi-GPU merge with the exchange fused into the merge kernels.

    Every rank exports its A and B shards (CUDA IPC); every rank maps all
    peers' shards once (peer access over NVLink 5 / NVSwitch) and runs
    mp_merge_pieces on its output slice S[floor(rN/P), floor((r+1)N/P)):
    the tile split searches and the tile loads read peer HBM directly -- no
    all_to_all, no staging buffer, two kernels per rank.  Each call is
    ordered across ranks on the GPU alone (_Flags): READY (every shard's
    producer has finished) before the merge, DONE (every peer has finished
    reading) after it, so the host never blocks and no barrier runs per
    call."""

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
        self._imported = []  # peer mappings this object holds (closed by close())
        for r, (la, lb, ea, eb, eav, ebv) in enumerate(recs):
            if r == self.comm.rank:
                ka, kb = a_local.data_ptr() if la else 0, b_local.data_ptr() if lb else 0
                va = a_vals.data_ptr() if a_vals is not None and la else None
                vb = b_vals.data_ptr() if b_vals is not None and lb else None
            else:
                ka, kb = _import(ea), _import(eb)
                va = _import(eav) if eav is not None else None
                vb = _import(ebv) if ebv is not None else None
                self._imported += [x for x in (ka, kb, va, vb) if x]
            self.pa.append((ka or None, va, la))
            self.pb.append((kb or None, vb, lb))
        self.na = sum(p[2] for p in self.pa)
        self.nb = sum(p[2] for p in self.pb)
        n, P, r = self.na + self.nb, self.comm.world, self.comm.rank
        self.o0, self.o1 = r * n // P, (r + 1) * n // P
        self._arr_a = N.pieces_array(self.pa)
        self._arr_b = N.pieces_array(self.pb)
        self.flags = _Flags(self.comm, a_local.device)
        self._imported += self.flags.imported

    def close(self):
        """Drop this object's peer mappings (mp_ipc_close; the library
        unmaps an allocation when its last importer closes it).  Call on
        every rank after the last call, once the streams are done."""
        for p in getattr(self, "_imported", []):
            N.check(N.lib.mp_ipc_close(p))
        self._imported = []

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown / library already gone
            pass

    def splits(self):
        """a_off of the merge path at this rank's slice ends (o0, o1), found
        by mp_pieces_partition over the mapped shards (device search, the
        kernels' own predicate)."""
        dev = self.a.device
        d = torch.tensor([self.o0, self.o1], dtype=torch.int64, device=dev)
        a = torch.empty(2, dtype=torch.int64, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        self.flags.arrive(_Flags.READY, range(self.comm.world), st)
        N.check(N.lib.mp_pieces_partition(self.kt, self._arr_a, len(self.pa), self._arr_b,
                                          len(self.pb), d.data_ptr(), 2, a.data_ptr(), st))
        self.flags.arrive(_Flags.DONE, range(self.comm.world), st)
        return a.tolist()

    def traffic(self):
        """Collective (every rank calls it).  Per rank r: the elements of r's
        output slice that live on other ranks' shards (r's NVLink-in, in
        keys: in_a + in_b), the elements of r's own shards that other ranks
        read (r's NVLink-out) and the elements r's HBM serves (its local
        reads, its peers' reads of its shards, its output writes) -- all
        from the actual split points (splits(), untimed bookkeeping)."""
        P = self.comm.world
        la = [p[2] for p in self.pa]
        lb = [p[2] for p in self.pb]
        sp = self.comm.all_gather_int(self.splits())
        sa = [sum(la[:r]) for r in range(P + 1)]
        sb = [sum(lb[:r]) for r in range(P + 1)]
        n = self.na + self.nb

        def ov(lo, hi, q, starts):
            return max(0, min(hi, starts[q + 1]) - max(lo, starts[q]))

        rng = []
        for r in range(P):
            a0, a1 = sp[r]
            rng.append((a0, a1, r * n // P - a0, (r + 1) * n // P - a1))
        res = []
        for r in range(P):
            a0, a1, b0, b1 = rng[r]
            own = ov(a0, a1, r, sa) + ov(b0, b1, r, sb)
            served = sum(ov(x[0], x[1], r, sa) + ov(x[2], x[3], r, sb)
                         for q, x in enumerate(rng))
            res.append({"in": (a1 - a0) + (b1 - b0) - own, "out": served - own,
                        "hbm_read": served, "hbm_write": (a1 - a0) + (b1 - b0),
                        "hbm": served + (a1 - a0) + (b1 - b0)})
        return res

    def __call__(self, out=None, out_vals=None):
        m = self.o1 - self.o0
        if out is None:
            out = torch.empty(m * (2 if self.kt == N.KEY_ELEMENT else 1),
                              dtype=self.a.dtype if self.kt != N.KEY_ELEMENT else torch.int64,
                              device=self.a.device)
        if out_vals is None and self.av is not None:
            out_vals = torch.empty(m, dtype=torch.uint32, device=self.a.device)
        st = torch.cuda.current_stream(self.a.device).cuda_stream
        ranks = range(self.comm.world)
        self.flags.arrive(_Flags.READY, ranks, st)
        N.check(N.lib.mp_merge_pieces(self.kt, self._arr_a, len(self.pa), self._arr_b,
                                      len(self.pb), self.o0, self.o1, out.data_ptr(),
                                      out_vals.data_ptr() if out_vals is not None else None,
                                      st))
        self.flags.arrive(_Flags.DONE, ranks, st)
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
    buffer, then ping/pong swap.  Each round is ordered among the pair's
    ranks on the GPU alone (_Flags READY before the merge, DONE after it:
    nobody overwrites a buffer a peer may still read).  Slice sizes are
    computed, not communicated: every rank knows every length (pass `lens`
    to skip the one host all_gather of the shard sizes)."""

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
        self._imported = []
        for r, (e0, e1) in enumerate(recs):
            if r == self.comm.rank:
                self.peer[r] = [self.buf[0].data_ptr(), self.buf[1].data_ptr()]
            else:
                self.peer[r] = [_import(e0), _import(e1)]
                self._imported += [x for x in self.peer[r] if x]
        self.flags = _Flags(self.comm, dev)
        self._imported += self.flags.imported
        self.scratch = None

    close = P2PMerger.close
    __del__ = P2PMerger.__del__

    @staticmethod
    def schedule(lens):
        """The rounds: for each round, (left ranks, right ranks, new lens) per
        rank group, and each rank's output range in its group's merge."""
        P = len(lens)
        rounds, h = [], 1
        while h < P:
            new_lens = list(lens)
            groups = []
            for s in range(0, P, 2 * h):
                L = list(range(s, min(s + h, P)))
                R = list(range(s + h, min(s + 2 * h, P)))
                if R:
                    owners = L + R
                    tot = sum(lens[q] for q in owners)
                    for k, q in enumerate(owners):
                        new_lens[q] = (k + 1) * tot // len(owners) - k * tot // len(owners)
                groups.append((L, R, list(lens)))
            rounds.append(groups)
            lens = new_lens
            h *= 2
        return rounds, lens

    def run(self, x_local: torch.Tensor, lens=None, trace=None):
        """Sort; returns this rank's slice of the sorted sequence.  With a
        list `trace`, each merge round appends (owners, k, o0, o1, splits)
        -- the actual split points of this rank's slice, searched over the
        round's mapped inputs (mp_pieces_partition) -- for sort_traffic()."""
        P, me = self.comm.world, self.comm.rank
        kt = self.kt
        n_me = n_keys(x_local, kt)
        if n_me > self.capacity:
            # buf[0] holds `capacity` keys and is mapped into every peer:
            # an overrun would corrupt memory the peers read
            raise ValueError(f"P2PSorter.run: shard of {n_me} keys exceeds the capacity "
                             f"{self.capacity} set at construction")
        if lens is None:
            lens = [x[0] for x in self.comm.all_gather_int([n_me])]
        elif len(lens) != P or lens[me] != n_me:
            raise ValueError("P2PSorter.run: lens must list every rank's shard size")
        stream = torch.cuda.current_stream(self.buf[0].device)
        st = stream.cuda_stream
        sb = N.lib.mp_sort_scratch_bytes(kt, 0, n_me)
        if self.scratch is None or self.scratch.numel() < max(sb, 16):
            self.scratch = torch.empty(max(sb, 16), dtype=torch.uint8, device=self.buf[0].device)
        N.check(N.lib.mp_sort_to(kt, x_local.data_ptr(), None, self.buf[0].data_ptr(), None,
                                 n_me, self.scratch.data_ptr(), self.scratch.numel(), st))
        rounds, final = self.schedule(lens)
        cur = 0
        for groups in rounds:
            L, R, glens = next(g for g in groups if me in g[0] + g[1])
            if R:
                owners = L + R
                k = owners.index(me)
                tot = sum(glens[q] for q in owners)
                o0, o1 = k * tot // len(owners), (k + 1) * tot // len(owners)
                if o1 - o0 > self.capacity:  # an equal split never exceeds the largest shard
                    raise ValueError("P2PSorter.run: round slice exceeds the capacity")
                pa = N.pieces_array([(self.peer[q][cur] if glens[q] else None, None, glens[q])
                                     for q in L])
                pb = N.pieces_array([(self.peer[q][cur] if glens[q] else None, None, glens[q])
                                     for q in R])
                self.flags.arrive(_Flags.READY, owners, st)
                if trace is not None:
                    dev = self.buf[0].device
                    d = torch.tensor([o0, o1], dtype=torch.int64, device=dev)
                    sp = torch.empty(2, dtype=torch.int64, device=dev)
                    N.check(N.lib.mp_pieces_partition(kt, pa, len(L), pb, len(R), d.data_ptr(),
                                                      2, sp.data_ptr(), st))
                    trace.append((owners, len(L), [glens[q] for q in owners], o0, o1, sp, d))
                N.check(N.lib.mp_merge_pieces(kt, pa, len(L), pb, len(R), o0, o1,
                                              self.buf[1 - cur].data_ptr(), None, st))
                self.flags.arrive(_Flags.DONE, owners, st)
            else:  # carried block: copy through so every rank sits in `1-cur`
                words = glens[me] * (2 if kt == N.KEY_ELEMENT else 1)
                self.buf[1 - cur][:words].copy_(self.buf[cur][:words])
                self.flags.gen += 2  # keep the generation in step with the paired ranks
                if trace is not None:
                    trace.append(None)
            cur = 1 - cur
        words = final[me] * (2 if kt == N.KEY_ELEMENT else 1)
        return self.buf[cur][:words]


def _overlap(lo, hi, s0, s1):
    return max(0, min(hi, s1) - max(lo, s0))


def sort_traffic(comm, trace, lens, run0=16384):
    """Collective.  Per-rank, per-phase element counts of one P2PSorter.run
    (from a traced run): phase 0 = the local sort (its algorithmic HBM
    passes: block sort + ceil(log2(n/run0)) rounds, each reading and writing
    every key once); phase k >= 1 = cross round k: NVLink-in (elements of my
    slice on other ranks), NVLink-out (elements of my block read by others),
    HBM (elements my HBM serves to me and my peers + my slice's writes).
    Returns (phases, final lens) with phases[k][r] = dict(in, out, hbm)."""
    P, me = comm.world, comm.rank
    rows = [None if t is None else (t[3], t[4]) + tuple(t[5].tolist()) for t in trace]
    groups = [None if t is None else (t[0], t[1], t[2]) for t in trace]
    allrows = [None] * P
    dist.all_gather_object(allrows, (rows, groups), group=comm.group)
    rounds, _ = P2PSorter.schedule(lens)

    def lens_at(k, r):  # rank r's block length entering round k
        return rounds[k][0][2][r] if rounds[k] else lens[r]

    phases = []
    local = []
    for r in range(P):
        w, passes = run0, 1
        while w < lens[r]:
            w, passes = 2 * w, passes + 1
        local.append({"in": 0, "out": 0, "hbm": 2 * lens[r] * passes})
    phases.append(local)
    for k in range(len(rounds)):
        ph = [{"in": 0, "out": 0, "hbm": 0} for _ in range(P)]
        # each rank's (a0, a1, b0, b1) in its group's A/B index spaces
        rng = {}
        for r in range(P):
            rws, gps = allrows[r]
            if rws[k] is None:  # carried block: a local copy
                ph[r]["hbm"] += 2 * lens_at(k, r)
                continue
            o0, o1, a0, a1 = rws[k]
            owners, nl, gl = gps[k]
            rng[r] = (owners, nl, gl, a0, a1, o0 - a0, o1 - a1)
        for r, (owners, nl, gl, a0, a1, b0, b1) in rng.items():
            # piece extents of every owner in the group's A (left) / B (right) space
            ext = {}
            s = 0
            for q, ln in zip(owners[:nl], gl[:nl]):
                ext[q] = ("a", s, s + ln)
                s += ln
            s = 0
            for q, ln in zip(owners[nl:], gl[nl:]):
                ext[q] = ("b", s, s + ln)
                s += ln
            for q in owners:
                side, s0, s1 = ext[q]
                got = _overlap(a0, a1, s0, s1) if side == "a" else _overlap(b0, b1, s0, s1)
                ph[q]["hbm"] += got          # q's HBM serves r's read
                if q != r:
                    ph[r]["in"] += got
                    ph[q]["out"] += got
            ph[r]["hbm"] += (a1 - a0) + (b1 - b0)  # r's slice written to its HBM
        phases.append(ph)
    return phases


def roofline_time(phases, key_bytes, hbm_gbs, nvl_gbs):
    """t_g = sum over phases of max(HBM_g / HBM peak,
    NVin_g / NVLink, NVout_g / NVLink); returns (max_g t_g in s, [t_g])."""
    P = len(phases[0])
    tg = []
    for g in range(P):
        t = 0.0
        for ph in phases:
            x = ph[g]
            t += max(x["hbm"] * key_bytes / (hbm_gbs * 1e9),
                     x["in"] * key_bytes / (nvl_gbs * 1e9),
                     x["out"] * key_bytes / (nvl_gbs * 1e9))
        tg.append(t)
    return max(tg), tg


def nvlink_probe(comm, device, mib=1024, reps=5):
    """Measured NVLink pull rate: every rank reads `mib` MiB from rank
    (r+1) % P's HBM into its own with SM vector loads (mp_peer_copy, the
    peer loader's access pattern), all ranks at once; CUDA events on the
    launching stream.  Returns (GB/s per rank, min over ranks).  On one GPU
    shared by several ranks it measures same-device IPC copies."""
    P, me = comm.world, comm.rank
    nbytes = mib << 20
    src = torch.empty(nbytes, dtype=torch.uint8, device=device)
    dst = torch.empty(nbytes, dtype=torch.uint8, device=device)
    src.fill_(me & 0xFF)
    recs = [None] * P
    dist.all_gather_object(recs, _export(src), group=comm.group)
    peer = _import(recs[(me + 1) % P]) if P > 1 else src.data_ptr()
    flags = _Flags(comm, device)
    st = torch.cuda.current_stream(device)
    ranks = range(P)
    rates = []
    for i in range(reps + 1):
        flags.arrive(_Flags.READY, ranks, st.cuda_stream)  # all ranks start together
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        N.check(N.lib.mp_peer_copy(dst.data_ptr(), peer, nbytes, st.cuda_stream))
        e1.record(st)
        flags.arrive(_Flags.DONE, ranks, st.cuda_stream)
        st.synchronize()
        if i:  # first pull warms the mapping
            rates.append(nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    if P > 1:
        N.check(N.lib.mp_ipc_close(peer))
    for x in flags.imported:
        N.check(N.lib.mp_ipc_close(x))
    import statistics
    mine = statistics.median(rates)
    allr = comm.all_gather_int([int(mine * 1000)])
    per_rank = [x[0] / 1000 for x in allr]
    return per_rank, min(per_rank)


# --------------------------------------------------------------------------
# one process, several GPUs: the shard-table C ABI (mp_multi_merge / _sort)
# --------------------------------------------------------------------------
def _shard_table(keys, vals, kt):
    rows = []
    for k, v in zip(keys, vals if vals is not None else [None] * len(keys)):
        if not k.is_cuda:
            raise ValueError("shards must be CUDA tensors")
        n = n_keys(k, kt)
        rows.append((k.device.index, k.data_ptr() if n else None,
                     v.data_ptr() if v is not None and n else None, n))
    return N.shards_array(rows), len(rows)


def multi_sort(shards, vals=None, key_type=None, streams=None):
    """Stable in-place sort of the sequence shards[0] ++ shards[1] ++ ...
    (CUDA tensors on any devices of this process, 1..16 of them; `vals`
    optional uint32 tensors alongside): afterwards shards[g] holds its slice
    of the sorted sequence (mp_multi_sort: local sorts, then Merge Path
    rounds between device groups over NVLink).  Blocking unless `streams`
    (one torch stream per shard) is given."""
    kt = key_type_of(shards[0], key_type)
    tab, n = _shard_table(shards, vals, kt)
    st = None
    if streams is not None:
        st = (C_void_p * n)(*[s.cuda_stream for s in streams])
    N.check(N.lib.mp_multi_sort(kt, tab, n, st))
    return shards


def multi_merge(a_shards, b_shards, out_shards, a_vals=None, b_vals=None, out_vals=None,
                key_type=None, streams=None):
    """Stable merge of A = a_shards[0] ++ ... and B = b_shards[0] ++ ...
    (ties: A first) into out_shards (their lengths sum to |A| + |B|); each
    output shard is computed on its own device, reading the inputs over
    NVLink (mp_multi_merge).  Blocking unless `streams` (one per output
    shard) is given."""
    kt = key_type_of(a_shards[0], key_type)
    ta, na = _shard_table(a_shards, a_vals, kt)
    tb, nb = _shard_table(b_shards, b_vals, kt)
    to, no = _shard_table(out_shards, out_vals, kt)
    st = None
    if streams is not None:
        st = (C_void_p * no)(*[s.cuda_stream for s in streams])
    N.check(N.lib.mp_multi_merge(kt, ta, na, tb, nb, to, no, st))
    return out_shards


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
# bench.py --gpus N (N > 1): one process per GPU over NCCL
# --------------------------------------------------------------------------
class _NoClock:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False

    def summary(self):
        return None


def _peaks():
    import json
    from pathlib import Path
    f = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    if f.exists():
        return float(json.loads(f.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _time_steps(step, steps, warmup, comm, red_dev, clock):
    """W untimed steps, then EXACTLY `steps` steps between a barrier +
    synchronize on both sides, timed with CUDA events on the launching
    stream; returns the max over ranks in ms and the launches counted."""
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier(group=comm.group)
    st = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    c0 = N.lib.mp_launch_count()
    with (clock or _NoClock)() as clk:
        e0.record(st)
        for _ in range(steps):
            step()
        e1.record(st)
        torch.cuda.synchronize()
    launches = N.lib.mp_launch_count() - c0
    dist.barrier(group=comm.group)
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=red_dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX, group=comm.group)
    return float(ms.item()), launches, clk.summary()


def _nvl(comm, dev, shrink):
    """The NVLink rate the roofline is computed against: measured here
    (nvlink_probe) -- ranks sharing one GPU (MP_BENCH_DEVICE) measure a
    same-device copy, which is said in the source field."""
    import os
    try:
        per, low = nvlink_probe(comm, dev, mib=max(16, 1024 >> shrink))
        shared = "MP_BENCH_DEVICE" in os.environ
        src = ("measured in this run: mp_peer_copy pull from rank (r+1)%P, all ranks at once"
               + (" (ranks share ONE GPU: same-device copy, not NVLink)" if shared else ""))
        return low, per, src
    except Exception as e:  # pragma: no cover
        return 900.0, None, f"spec 900 GB/s per direction (probe failed: {e})"


def bench_distributed(args, cfg, ws, rank, local, clock=None):
    """A merge config at N GPUs.  Configs 2/3 (weak scaling): each rank
    holds the config's |A| and |B| as its shard of globally sorted A and B
    (SplitMix64 counter generator at the rank's global offsets, then sorted
    across the ranks with sharded_sort -- untimed).  Config 5 (strong
    scaling): the fixed 2^31 + 2^31 f32 inputs sharded contiguously.  A
    timed step is one P2PMerger call: each rank merges its output slice
    straight from the mapped shards (NVLink pull fused into the tile loads),
    ordered across ranks by stream flags only.  Max over ranks."""
    import os
    import time
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    comm = _Comm()
    kt = {"u32": N.KEY_U32, "i32": N.KEY_I32, "f32": N.KEY_F32, "u64": N.KEY_U64,
          "i64": N.KEY_I64}[cfg["key"]]
    dt = {"u32": torch.uint32, "i32": torch.int32, "f32": torch.float32,
          "u64": torch.uint64, "i64": torch.int64}[cfg["key"]]
    st = torch.cuda.current_stream().cuda_stream

    def gen(kind, seed, n, first):
        x = torch.empty(n, dtype=dt, device=dev)
        N.check(N.lib.mp_generate(kind, seed, first, n, x.data_ptr(), st))
        return x

    # MP_BENCH_SCALE=k shrinks the sizes by 2^k (multi-rank smoke tests on
    # a one-GPU box)
    shrink = int(os.environ.get("MP_BENCH_SCALE", "0"))
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
        la = [x[0] for x in comm.all_gather_int([a.numel()])]
        lb = [x[0] for x in comm.all_gather_int([b.numel()])]
        av = (torch.arange(a.numel(), dtype=torch.int64, device=dev) + sum(la[:rank])
              ).to(torch.int32).view(torch.uint32)
        bv = ((torch.arange(b.numel(), dtype=torch.int64, device=dev) + sum(lb[:rank]))
              | (1 << 31)).to(torch.int32).view(torch.uint32)
    merger = P2PMerger(a, b, av, bv, key_type=kt)  # IPC mappings + flags, once (untimed)
    out = torch.empty(merger.o1 - merger.o0, dtype=dt, device=dev)
    outv = torch.empty(out.numel(), dtype=torch.uint32, device=dev) if av is not None else None
    step = lambda: merger(out, outv)  # noqa: E731
    ms, launches, clk = _time_steps(step, args.steps, args.warmup, comm, red_dev, clock)
    total = (NA + NB) if strong else (na + nb) * ws
    value = total * args.steps / (ms / 1e3)
    # traffic from the actual split points, HBM + NVLink roofline
    tr = merger.traffic()
    hbm, hbm_src = _peaks()
    nvl, nvl_per, nvl_src = _nvl(comm, dev, shrink)
    ks = a.element_size() + (4 if av is not None else 0)  # key (+ value) bytes
    t_roof, tg = roofline_time([tr], ks, hbm, nvl)
    # e2e through the public API with host buffers: H2D of this rank's
    # shards, the sharded merge, D2H of its output slice (wall clock, max
    # over ranks)
    ha, hb = a.cpu().pin_memory(), b.cpu().pin_memory()
    hav = av.cpu().pin_memory() if av is not None else None
    hbv = bv.cpu().pin_memory() if bv is not None else None
    ho = torch.empty(out.numel(), dtype=dt).pin_memory()
    hov = torch.empty(out.numel(), dtype=torch.uint32).pin_memory() if av is not None else None
    e2e_steps = max(1, min(args.steps, getattr(args, "e2e_steps", 3)))
    torch.cuda.synchronize()
    dist.barrier()
    t = time.perf_counter()
    for _ in range(e2e_steps):
        a.copy_(ha, non_blocking=True)  # H2D into the mapped shards
        b.copy_(hb, non_blocking=True)
        if hav is not None:
            av.copy_(hav, non_blocking=True)
            bv.copy_(hbv, non_blocking=True)
        merger(out, outv)
        ho.copy_(out, non_blocking=True)
        if hov is not None:
            hov.copy_(outv, non_blocking=True)
    torch.cuda.synchronize()
    el = torch.tensor([time.perf_counter() - t], dtype=torch.float64, device=red_dev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    merger.close()
    return {
        "metric": "merged elements/s", "value": value, "unit": "elements/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": cfg["key"],
        "data": "synthetic: SplitMix64 counter generator, globally sorted with sharded_sort",
        "config": {"workload": cfg["desc"] + (f"; sharded over {ws} GPUs" if strong else
                                             f" per GPU; global |A|={NA * ws} |B|={NB * ws}"),
                   "parallelism": f"merge-path diagonal split over {ws} GPUs (NVLink pull "
                                  "fused into the merge kernels via CUDA IPC; stream-flag "
                                  "ordering, no host sync per step)",
                   "l2": "inputs+output larger than L2 (no flush needed)"},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm+nvlink", "unit": "elements/s", "achieved": value,
                     "peak": total / t_roof, "frac": value / (total / t_roof),
                     "traffic": None,
                     "model": "N / max_g max(HBM_g/hbm_gbs, NVin_g/nvlink_gbs, NVout_g/nvlink_gbs)"
                              " from the actual split points",
                     "hbm_gbs": hbm, "hbm_source": hbm_src, "nvlink_gbs": nvl,
                     "nvlink_source": nvl_src, "nvlink_gbs_per_rank": nvl_per,
                     "t_g_ms": [x * 1e3 for x in tg]},
        "nvlink": {"in_bytes_per_rank": [x["in"] * ks for x in tr],
                   "out_bytes_per_rank": [x["out"] * ks for x in tr],
                   "hbm_bytes_per_rank": [x["hbm"] * ks for x in tr]},
        "clocks": clk,
        "e2e": {"value": total * e2e_steps / float(el.item()), "unit": "elements/s",
                "h2d_bytes_per_step": (na + nb) * ks, "d2h_bytes_per_step": out.numel() * ks},
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
    comm = _Comm()
    shrink = int(os.environ.get("MP_BENCH_SCALE", "0"))
    n = cfg["n"] >> shrink
    lo, hi = rank * n // ws, (rank + 1) * n // ws
    lens = [(r + 1) * n // ws - r * n // ws for r in range(ws)]
    x = torch.empty(hi - lo, dtype=torch.uint32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    N.check(N.lib.mp_generate(cfg["gen"][0], 4, lo, hi - lo, x.data_ptr(), st))
    sorter = P2PSorter(max(lens) + 1, torch.uint32, N.KEY_U32)
    red_dev = dev if dist.get_backend() == "nccl" else torch.device("cpu")
    ms, launches, clk = _time_steps(lambda: sorter.run(x, lens), args.steps, args.warmup,
                                    comm, red_dev, clock)
    # traced run (untimed): the actual split points of every round
    trace = []
    sorter.run(x, lens, trace=trace)
    torch.cuda.synchronize()
    phases = sort_traffic(comm, trace, lens)
    hbm, hbm_src = _peaks()
    nvl, nvl_per, nvl_src = _nvl(comm, dev, shrink)
    t_roof, tg = roofline_time(phases, 4, hbm, nvl)
    # e2e: pinned host shard -> device, sort, sorted slice back to the host
    hx = x.cpu().pin_memory()
    _, final = P2PSorter.schedule(lens)
    ho = torch.empty(final[rank], dtype=torch.uint32).pin_memory()
    e2e_steps = max(1, min(args.steps, getattr(args, "e2e_steps", 3)))
    torch.cuda.synchronize()
    dist.barrier()
    t = time.perf_counter()
    for _ in range(e2e_steps):
        x.copy_(hx, non_blocking=True)
        ho.copy_(sorter.run(x, lens), non_blocking=True)
    torch.cuda.synchronize()
    el = torch.tensor([time.perf_counter() - t], dtype=torch.float64, device=red_dev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    sorter.close()
    value = n * args.steps / (ms / 1e3)
    return {
        "metric": "merge-sort keys/s", "value": value, "unit": "keys/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32",
        "data": "synthetic: SplitMix64 counter generator, seed 4",
        "config": {"workload": cfg["desc"] + f"; {ws} GPUs, 1/{ws} shard each",
                   "parallelism": f"local sort + {(ws - 1).bit_length()} cross-GPU Merge Path "
                                  "rounds, NVLink pull fused into the merge (CUDA IPC), "
                                  "stream-flag ordering",
                   "l2": "inputs+output larger than L2 (no flush needed)"},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm+nvlink", "unit": "keys/s", "achieved": value,
                     "peak": n / t_roof, "frac": value / (n / t_roof), "traffic": None,
                     "model": "N / max_g sum_phases max(HBM_g/hbm_gbs, NVin_g/nvlink_gbs, "
                              "NVout_g/nvlink_gbs); local sort = (1 + rounds) passes x 8 B/key, "
                              "cross rounds from the traced split points",
                     "hbm_gbs": hbm, "hbm_source": hbm_src, "nvlink_gbs": nvl,
                     "nvlink_source": nvl_src, "nvlink_gbs_per_rank": nvl_per,
                     "t_g_ms": [t * 1e3 for t in tg]},
        "nvlink": {"in_bytes_per_rank": [sum(ph[r]["in"] for ph in phases) * 4
                                         for r in range(ws)],
                   "out_bytes_per_rank": [sum(ph[r]["out"] for ph in phases) * 4
                                          for r in range(ws)]},
        "clocks": clk,
        "e2e": {"value": n * e2e_steps / float(el.item()), "unit": "keys/s",
                "h2d_bytes_per_step": (hi - lo) * 4, "d2h_bytes_per_step": final[rank] * 4},
    }
