// mp_multi.cuh -- single-process multi-GPU merge and sort over a shard table
// {device, keys, vals, len}[P] (include/mergepath_b200.h mp_multi_merge /
// mp_multi_sort): the C-ABI form of the per-GPU path that multigpu.py runs
// with one process per GPU.  Included by mp_capi.cu after PiecesOp.
//
// Every output shard g is produced on its own device by the piece-list merge
// (mp_pieces.cuh): its tile split points are searched over the virtual index
// spaces of A and B and its windows are read straight from whichever device
// holds them (peer access over NVLink / NVSwitch, LSU loads for remote
// windows) -- no staging copy, no collective.  The sort is the local sort of
// every shard followed by ceil(log2 P) rounds of such merges between rank
// groups (left group = A, so it stays stable w.r.t. the input order;
// sort.hpp:71-128 at GPU granularity), ping-ponging between the shard and
// one scratch buffer per shard.
//
// Ordering is stream-ordered across devices with events only: a "fence"
// records an event on every participating stream and makes every stream
// wait for all of them, so a phase starts after every stream finished the
// previous one (inputs written, peers done reading).  The host never waits,
// except in the blocking form (streams == NULL) at entry and exit.
#pragma once

namespace {

int cuda_copy(void *dst, const void *src, size_t bytes, cudaStream_t s) {
  MP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
  return MP_OK;
}

struct MultiCtx {
  int P = 0;
  std::vector<int> dev;
  std::vector<cudaStream_t> st;
  std::vector<cudaEvent_t> ev;
  bool own = false;  // internal streams (blocking call)

  // x[0..n): the shards whose streams take part; `others` = devices that
  // only hold inputs (synchronised in the blocking form, peer access on)
  int setup(const mp_shard *x, int n, void *const *streams, std::vector<int> others = {}) {
    P = n;
    dev.resize(n);
    st.resize(n);
    ev.assign(n, nullptr);
    own = streams == nullptr;
    for (int g = 0; g < n; ++g) {
      dev[g] = x[g].device;
      DeviceScope ds(dev[g]);
      if (ds.err != cudaSuccess)
        return cuda_fail(ds.err, "multi: cudaSetDevice");
      if (own) {
        MP_CUDA(cudaDeviceSynchronize());  // inputs complete (blocking form)
        MP_CUDA(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
      } else {
        st[g] = static_cast<cudaStream_t>(streams[g]);
      }
      MP_CUDA(cudaEventCreateWithFlags(&ev[g], cudaEventDisableTiming));
    }
    for (int d : others) {
      if (own) {
        DeviceScope ds(d);
        MP_CUDA(cudaDeviceSynchronize());
      }
    }
    // peer access from every participating device to every other device
    std::vector<int> all(dev);
    all.insert(all.end(), others.begin(), others.end());
    for (int g = 0; g < n; ++g)
      for (int h : all) {
        if (dev[g] == h)
          continue;
        int ok = 0;
        MP_CUDA(cudaDeviceCanAccessPeer(&ok, dev[g], h));
        if (!ok)
          return fail(MP_ERR_UNSUPPORTED, "multi: device %d cannot access device %d",
                      dev[g], h);
        DeviceScope ds(dev[g]);
        const cudaError_t e = cudaDeviceEnablePeerAccess(h, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled)
          cudaGetLastError();
        else if (e != cudaSuccess)
          return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      }
    return MP_OK;
  }

  // every stream waits for the work enqueued so far on every stream
  int fence() {
    for (int g = 0; g < P; ++g) {
      DeviceScope ds(dev[g]);
      MP_CUDA(cudaEventRecord(ev[g], st[g]));
    }
    for (int g = 0; g < P; ++g) {
      DeviceScope ds(dev[g]);
      for (int h = 0; h < P; ++h)
        if (h != g)
          MP_CUDA(cudaStreamWaitEvent(st[g], ev[h], 0));
    }
    return MP_OK;
  }

  int finish() {
    int rc = MP_OK;
    for (int g = 0; g < P; ++g) {
      DeviceScope ds(dev[g]);
      if (own && st[g]) {
        if (cudaStreamSynchronize(st[g]) != cudaSuccess && rc == MP_OK)
          rc = cuda_fail(cudaGetLastError(), "multi: cudaStreamSynchronize");
        cudaStreamDestroy(st[g]);
      }
      if (ev[g])
        cudaEventDestroy(ev[g]);
    }
    return rc;
  }
};

// values ride along when any shard of the table carries them (an empty
// shard may have no value pointer)
bool any_vals(const mp_shard *x, int n) {
  for (int g = 0; g < n; ++g)
    if (x[g].vals)
      return true;
  return false;
}

int check_shards(const mp_shard *x, int n, const char *what, bool vals_all) {
  if (n < 1 || n > kMaxPieces)
    return fail(MP_ERR_INVALID, "multi: 1..%d %s shards", kMaxPieces, what);
  int ndev = 0;
  MP_CUDA(cudaGetDeviceCount(&ndev));
  for (int g = 0; g < n; ++g) {
    if (x[g].device < 0 || x[g].device >= ndev)
      return fail(MP_ERR_INVALID, "multi: %s shard %d on no device (%d)", what, g,
                  x[g].device);
    if (x[g].len && !x[g].keys)
      return fail(MP_ERR_INVALID, "multi: %s shard %d has no keys", what, g);
    if (vals_all && x[g].len && !x[g].vals)
      return fail(MP_ERR_INVALID, "multi: %s shard %d has no values", what, g);
  }
  return MP_OK;
}

template <class KT> struct MultiMergeOp {
  static int run(const mp_shard *a, int na, const mp_shard *b, int nb, const mp_shard *o,
                 int no, void *const *streams) {
    if (no < 1 || no > kMaxPieces)
      return fail(MP_ERR_INVALID, "multi: 1..%d out shards", kMaxPieces);
    const bool vals = any_vals(o, no);
    if (int rc = check_shards(a, na, "A", vals))
      return rc;
    if (int rc = check_shards(b, nb, "B", vals))
      return rc;
    if (int rc = check_shards(o, no, "out", vals))
      return rc;
    uint64_t n = 0, m = 0;
    for (int g = 0; g < na; ++g)
      n += a[g].len;
    for (int g = 0; g < nb; ++g)
      n += b[g].len;
    for (int g = 0; g < no; ++g)
      m += o[g].len;
    if (m != n)  // parallel.hpp:155-156 (output size must equal |A| + |B|)
      return fail(MP_ERR_INVALID, "multi_merge: output shards hold %llu, inputs %llu",
                  (unsigned long long)m, (unsigned long long)n);
    std::vector<mp_piece> pa(na), pb(nb);
    for (int g = 0; g < na; ++g)
      pa[g] = {a[g].keys, a[g].vals, a[g].len};
    for (int g = 0; g < nb; ++g)
      pb[g] = {b[g].keys, b[g].vals, b[g].len};
    std::vector<int> in_devs;
    for (int g = 0; g < na; ++g)
      in_devs.push_back(a[g].device);
    for (int g = 0; g < nb; ++g)
      in_devs.push_back(b[g].device);
    MultiCtx c;
    int rc = c.setup(o, no, streams, in_devs);
    if (rc == MP_OK)
      rc = c.fence();  // every input producer before any merge
    uint64_t o0 = 0;
    for (int g = 0; g < no && rc == MP_OK; ++g) {
      DeviceScope ds(o[g].device);
      rc = PiecesOp<KT>::run(pa.data(), na, pb.data(), nb, o0, o0 + o[g].len, o[g].keys,
                             o[g].vals, c.st[g]);
      o0 += o[g].len;
    }
    if (rc == MP_OK)
      rc = c.fence();  // every merge before later work on any stream
    const int rc2 = c.finish();
    return rc ? rc : rc2;
  }
};

template <class KT> struct MultiSortOp {
  static int run(const mp_shard *x, int P, void *const *streams) {
    using T = typename KT::T;
    if (P < 1 || P > kMaxPieces)
      return fail(MP_ERR_INVALID, "multi: 1..%d sort shards", kMaxPieces);
    const bool vals = any_vals(x, P);
    if (int rc = check_shards(x, P, "sort", vals))
      return rc;
    if (vals && KT::kind == kElement)
      return fail(MP_ERR_UNSUPPORTED, "ELEMENT keys carry their own tag");
    MultiCtx c;
    int rc = c.setup(x, P, streams);
    if (rc == MP_OK)
      rc = c.fence();
    // scratch per shard: the ping-pong partner (keys + values)
    std::vector<ScratchGuard> tmp(P);
    std::vector<T *> buf[2];
    std::vector<uint32_t *> vbuf[2];
    for (int k = 0; k < 2; ++k) {
      buf[k].assign(P, nullptr);
      vbuf[k].assign(P, nullptr);
    }
    for (int g = 0; g < P && rc == MP_OK; ++g) {
      DeviceScope ds(x[g].device);
      const uint64_t len = x[g].len;
      const uint64_t kb = (len * sizeof(T) + 255) & ~uint64_t(255);
      rc = alloc_scratch(tmp[g], kb + (vals ? len * 4 : 0), c.st[g]);
      if (rc)
        break;
      buf[0][g] = static_cast<T *>(x[g].keys);
      vbuf[0][g] = x[g].vals;
      buf[1][g] = static_cast<T *>(tmp[g].p);
      vbuf[1][g] = vals ? reinterpret_cast<uint32_t *>(static_cast<char *>(tmp[g].p) + kb)
                        : nullptr;
      // local sort of the shard, in place (stable; sort.hpp:132-148)
      if (len > 1)
        rc = SortOp<KT>::run(x[g].keys, x[g].vals, x[g].keys, x[g].vals, len, nullptr, 0,
                             c.st[g]);
    }
    int cur = 0;
    for (int h = 1; h < P && rc == MP_OK; h *= 2) {
      rc = c.fence();  // every block of this round complete; peers done with the other buffer
      for (int g = 0; g < P && rc == MP_OK; ++g) {
        const int s0 = (g / (2 * h)) * 2 * h;
        const int l0 = s0, l1 = std::min(s0 + h, P), r0 = l1, r1 = std::min(s0 + 2 * h, P);
        DeviceScope ds(x[g].device);
        if (r0 >= r1) {  // unpaired block: carried (sort.hpp:98-100)
          if (x[g].len)
            rc = cuda_copy(buf[1 - cur][g], buf[cur][g], x[g].len * sizeof(T), c.st[g]);
          if (rc == MP_OK && vals && x[g].len)
            rc = cuda_copy(vbuf[1 - cur][g], vbuf[cur][g], x[g].len * 4, c.st[g]);
          continue;
        }
        std::vector<mp_piece> pa, pb;
        for (int q = l0; q < l1; ++q)
          pa.push_back({buf[cur][q], vbuf[cur][q], x[q].len});
        for (int q = r0; q < r1; ++q)
          pb.push_back({buf[cur][q], vbuf[cur][q], x[q].len});
        // shard g keeps its own length: its slice of the group's output
        uint64_t o0 = 0;
        for (int q = l0; q < g; ++q)
          o0 += x[q].len;
        if (x[g].len)
          rc = PiecesOp<KT>::run(pa.data(), static_cast<int>(pa.size()), pb.data(),
                                 static_cast<int>(pb.size()), o0, o0 + x[g].len,
                                 buf[1 - cur][g], vals ? vbuf[1 - cur][g] : nullptr,
                                 c.st[g]);
      }
      cur = 1 - cur;
    }
    if (rc == MP_OK)
      rc = c.fence();
    if (cur == 1)  // the result sits in the scratch buffers: copy back
      for (int g = 0; g < P && rc == MP_OK; ++g) {
        DeviceScope ds(x[g].device);
        if (x[g].len)
          rc = cuda_copy(buf[0][g], buf[1][g], x[g].len * sizeof(T), c.st[g]);
        if (rc == MP_OK && vals && x[g].len)
          rc = cuda_copy(vbuf[0][g], vbuf[1][g], x[g].len * 4, c.st[g]);
      }
    for (int g = 0; g < P; ++g) {  // scratch freed on its own stream, after the copies
      DeviceScope ds(x[g].device);
      if (tmp[g].p)
        cudaFreeAsync(tmp[g].p, tmp[g].s);
      tmp[g].p = nullptr;
    }
    const int rc2 = c.finish();
    return rc ? rc : rc2;
  }
};

}  // namespace
