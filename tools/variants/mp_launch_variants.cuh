// mp_launch_variants.cuh -- measured-slower variants taken out of the product build
// (round 2).  Kept for reference and for A/B experiments: NOT compiled into
// libmergepath_b200.so.  Each block is headed by what it was and the B200
// measurement that retired it; it needs the product headers
// (paper_1406_2628_b200/csrc/) to compile.
#pragma once

// ===== PDL launches (MP_PDL=1) and the K1 || K2 side-stream overlap (MP_OVERLAP_CHUNKS) =====
// Launch with programmatic dependent launch (mp_common.cuh pdl_*): the
// kernel may become resident while the previous kernel of the stream drains
// and waits for it in pdl_wait().  Opt-in (MP_PDL=1): B200 A/B, config 2
// 0.650 vs 0.650 ms, config 4 31.16 vs 30.90 ms (the waiting CTAs of the
// next kernel sit in the previous one's last wave).
bool pdl_env() {
  static const bool b = [] {
    const char *e = std::getenv("MP_PDL");
    return e && std::strcmp(e, "1") == 0;
  }();
  return b;
}
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, uint32_t smem,
                       cudaStream_t s, Args &&...args) {
  if (!pdl_env()) {
    kern<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}



// ---- K1 || K2 overlap -------------------------------------------------------
// K1 (split search) is latency-bound: dependent DRAM probes, few bytes.  K2
// (tile merge) is HBM-bound.  Cut the tiles into chunks: the split points of
// chunk 0 are computed on the caller's stream, those of chunks 1.. on a
// high-priority side stream while chunk 0.. merge, so only chunk 0's search
// latency stays on the critical path.  Fork/join by events (graph-capturable).
constexpr int kOverlapChunks = 8;

struct SideStream {
  bool init = false;
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr;
  cudaEvent_t ev[kOverlapChunks] = {};
  int setup() {
    if (init)
      return MP_OK;
    int least = 0, greatest = 0;
    MP_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    MP_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, greatest));
    MP_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    for (auto &e : ev)
      MP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    init = true;
    return MP_OK;
  }
};

SideStream &side_stream() {
  thread_local SideStream ss[64];
  int dev = 0;
  cudaGetDevice(&dev);
  return ss[dev & 63];
}

// split(lo, hi, stream) fills split entries [lo, hi) of E; tile(t0, t1,
// stream) merges tiles [t0, t1) and reads entries [t0, t1] (< E).
template <class SplitFn, class TileFn>
int run_overlapped(uint64_t tiles, uint64_t E, SplitFn split, TileFn tile,
                   cudaStream_t s) {
  // Measured on B200 (round 1): the side-stream K1 chunks steal SM slots
  // from K2 and the step got slower, so the overlap is opt-in
  // (MP_OVERLAP_CHUNKS=2..8); the persistent SPM kernel removes K1 instead.
  static const int env_chunks = [] {
    const char *e = std::getenv("MP_OVERLAP_CHUNKS");
    const int v = e ? std::atoi(e) : 1;
    return v < 1 ? 1 : (v > kOverlapChunks ? kOverlapChunks : v);
  }();
  const int C = tiles >= 4096 ? env_chunks : 1;
  if (C == 1) {
    if (int rc = split(0, E, s))
      return rc;
    return tile(0, tiles, s);
  }
  SideStream &ss = side_stream();
  if (int rc = ss.setup())
    return rc;
  uint64_t T[kOverlapChunks + 1], B[kOverlapChunks + 1];
  for (int c = 0; c <= C; ++c) {
    T[c] = c * tiles / C;
    B[c] = c == 0 ? 0 : (c == C ? E : T[c] + 1);
  }
  if (int rc = split(B[0], B[1], s))
    return rc;
  MP_CUDA(cudaEventRecord(ss.fork, s));
  MP_CUDA(cudaStreamWaitEvent(ss.side, ss.fork, 0));
  for (int c = 1; c < C; ++c) {
    if (int rc = split(B[c], B[c + 1], ss.side))
      return rc;
    MP_CUDA(cudaEventRecord(ss.ev[c], ss.side));
  }
  for (int c = 0; c < C; ++c) {
    if (c > 0)
      MP_CUDA(cudaStreamWaitEvent(s, ss.ev[c], 0));
    if (int rc = tile(T[c], T[c + 1], s))
      return rc;
  }
  return MP_OK;
}

// ---- K2s: persistent streaming SPM merge (no global split pass) ----------
template <class KT> struct SpmShape;
template <> struct SpmShape<KeyU32> { static constexpr int NT = 256, VT = 15, CH = 1024, SLOTS = 8; };
template <> struct SpmShape<KeyI32> : SpmShape<KeyU32> {};
template <> struct SpmShape<KeyF32> : SpmShape<KeyU32> {};
template <> struct SpmShape<KeyU64> { static constexpr int NT = 256, VT = 11, CH = 512, SLOTS = 8; };
template <> struct SpmShape<KeyI64> : SpmShape<KeyU64> {};
template <> struct SpmShape<KeyElement> { static constexpr int NT = 256, VT = 7, CH = 256, SLOTS = 8; };

template <int NT_, int VT_, int CH_, int SLOTS_> struct SpmShapeX {
  static constexpr int NT = NT_, VT = VT_, CH = CH_, SLOTS = SLOTS_;
};

template <class KT, class Sh = SpmShape<KT>>
int spm_merge_shape(const void *a, uint64_t na, const void *b, uint64_t nb,
                    void *out, cudaStream_t s);

// tuning hook: MP_SPM_SHAPE=1..3 selects alternative ring geometries for
// 4-byte keys (A/B experiments); 0 = default
template <class KT>
int spm_merge(const void *a, uint64_t na, const void *b, uint64_t nb,
              void *out, cudaStream_t s) {
  static const int shape = [] {
    const char *e = std::getenv("MP_SPM_SHAPE");
    return e ? std::atoi(e) : 0;
  }();
  if constexpr (sizeof(typename KT::T) == 4) {
    if (shape == 1)
      return spm_merge_shape<KT, SpmShapeX<256, 15, 512, 16>>(a, na, b, nb, out, s);
    if (shape == 2)
      return spm_merge_shape<KT, SpmShapeX<256, 15, 1024, 16>>(a, na, b, nb, out, s);
    if (shape == 3)
      return spm_merge_shape<KT, SpmShapeX<512, 15, 1024, 16>>(a, na, b, nb, out, s);
  }
  return spm_merge_shape<KT>(a, na, b, nb, out, s);
}

template <class KT, class Sh>
int spm_merge_shape(const void *a, uint64_t na, const void *b, uint64_t nb,
                    void *out, cudaStream_t s) {
  using T = typename KT::T;
  using Cfg = SpmCfg<KT, Sh::NT, Sh::VT, Sh::CH, Sh::SLOTS>;
  auto kern = spm_merge_kernel<KT, Sh::NT, Sh::VT, Sh::CH, Sh::SLOTS>;
  static thread_local int grid_cache[64] = {};
  int dev = 0;
  MP_CUDA(cudaGetDevice(&dev));
  int &G = grid_cache[dev & 63];
  if (G == 0) {
    MP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(Cfg::bytes)));
    int sms = 0, per_sm = 0;
    MP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Sh::NT + 32,
                                                          Cfg::bytes));
    G = sms * (per_sm > 0 ? per_sm : 1);
  }
  const uint64_t n = na + nb;
  const uint64_t want = cdiv(n, 4ull * Cfg::NV);  // >= 4 windows per CTA
  const unsigned grid = static_cast<unsigned>(want < uint64_t(G) ? want : G);
  kern<<<grid ? grid : 1, Sh::NT + 32, Cfg::bytes, s>>>(
      static_cast<const T *>(a), na, static_cast<const T *>(b), nb,
      static_cast<T *>(out));
  MP_LAUNCHED("spm_merge_kernel");
  return MP_OK;
}

// Which engine a plain merge uses.  Default: the tile engine (K1 + K2).
// MP_MERGE_ENGINE=spm selects the persistent streaming SPM kernel for large
// key-only merges into a 16 B-aligned output.  Measured on B200 (round 1,
// tools/spm_check.py): bit-exact but 2.3x slower than K1+K2 -- one CTA's
// rings keep only ~17 KB per stream in flight, while 8 independent tile
// CTAs per SM keep ~120 KB in flight.
inline bool use_spm(uint64_t n, const void *out) {
  static const bool spm = [] {
    const char *e = std::getenv("MP_MERGE_ENGINE");
    return e && std::strcmp(e, "spm") == 0;
  }();
  return spm && n >= (1ull << 20) &&
         (reinterpret_cast<uintptr_t>(out) & 15) == 0;
}


// ===== PDL device hooks (mp_common.cuh) =====


// Programmatic dependent launch (PDL).  A kernel launched with the
// programmatic-stream-serialization attribute may become resident before
// the previous kernel in its stream has finished; pdl_wait() (griddepcontrol
// .wait) blocks until that kernel has completed and its memory is visible,
// and is a no-op for a normal launch.  pdl_launch_dependents() lets the next
// such kernel launch once every CTA of this grid has started.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ===== L2 evict_first bulk copies (MP_BULK_EVICT_FIRST) =====
// MP_BULK_EVICT_FIRST (compile-time A/B): the streamed windows and tiles
// carry an L2 evict_first policy (createpolicy + .L2::cache_hint).  B200:
// config 2 0.650 -> 0.650/0.678 ms, config 5 5.38 -> 5.42 ms, config 4
// 30.86 -> 30.96 ms -- no gain, off.
#ifndef MP_BULK_EVICT_FIRST
#define MP_BULK_EVICT_FIRST 0
#endif
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

