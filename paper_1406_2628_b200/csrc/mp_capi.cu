// mp_capi.cu -- the extern "C" boundary (include/mergepath_b200.h) and the
// host-side launch logic for the Merge Path kernels.
//
// Every entry point validates its arguments the way the reference does
// (invalid_argument conditions -> MP_ERR_INVALID), dispatches the key type to
// a kernel template instantiation, launches on the caller's stream and maps
// CUDA failures to status codes.  There is no CPU fallback: without a CUDA
// device every call fails with MP_ERR_CUDA.

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <utility>
#include <mutex>
#include <string>

#include "../../include/mergepath_b200.h"
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <thread>
#include <tuple>
#include <vector>

#include "mp_kernels.cuh"
#include "mp_pieces.cuh"
#include "mp_bsort.cuh"
#include "mp_quad.cuh"

namespace {

using namespace mpb;

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char *what) {
  return fail(e == cudaErrorMemoryAllocation ? MP_ERR_OOM : MP_ERR_CUDA,
              "%s: %s", what, cudaGetErrorString(e));
}

#define MP_CUDA(x)                                                             \
  do {                                                                         \
    const cudaError_t e_ = (x);                                                \
    if (e_ != cudaSuccess)                                                     \
      return cuda_fail(e_, #x);                                                \
  } while (0)

// Every kernel launch of the library is followed by MP_LAUNCHED, which also
// counts it (mp_launch_count: the bench's gpu_launches is this counter).
std::atomic<uint64_t> g_launches{0};

#define MP_LAUNCHED(what)                                                      \
  do {                                                                         \
    g_launches.fetch_add(1, std::memory_order_relaxed);                        \
    const cudaError_t e_ = cudaGetLastError();                                 \
    if (e_ != cudaSuccess)                                                     \
      return cuda_fail(e_, what);                                              \
  } while (0)

// Stream-ordered scratch from a library-private memory pool per device (not
// the device's default pool, which torch and the caller may share): the pool
// keeps its memory between calls (release threshold = max) so repeated calls
// do not hit the driver allocator; mp_release() trims it.
cudaMemPool_t g_pools[64] = {};

cudaMemPool_t lib_pool(int dev) {
  static std::once_flag once[64];
  if (dev < 0 || dev >= 64)
    return nullptr;
  std::call_once(once[dev], [dev] {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      g_pools[dev] = pool;
    } else {
      cudaGetLastError();
    }
  });
  return g_pools[dev];
}

struct ScratchGuard {  // frees a stream-ordered allocation on scope exit
  void *p = nullptr;
  cudaStream_t s = nullptr;
  ~ScratchGuard() {
    if (p)
      cudaFreeAsync(p, s);
  }
};

int alloc_scratch(ScratchGuard &g, size_t bytes, cudaStream_t s) {
  int dev = 0;
  MP_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool = lib_pool(dev);
  g.s = s;
  const cudaError_t e =
      pool ? cudaMallocFromPoolAsync(&g.p, bytes ? bytes : 16, pool, s)
           : cudaMallocAsync(&g.p, bytes ? bytes : 16, s);
  if (e != cudaSuccess) {
    g.p = nullptr;
    return cuda_fail(e, "cudaMallocAsync(scratch)");
  }
  return MP_OK;
}

struct DeviceScope {  // restores the caller's current device
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    err = cudaSetDevice(dev);
  }
  ~DeviceScope() {
    if (prev >= 0)
      cudaSetDevice(prev);
  }
};

uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Allocation holding p: cuMemGetAddressRange through the runtime's driver
// entry point (no link-time dependency on libcuda).  false if unknown.
bool alloc_range(const void *p, uintptr_t *base, size_t *size) {
  using GetRange = int (*)(unsigned long long *, size_t *, unsigned long long);
  static GetRange get_range = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      fn = nullptr;
    }
    return reinterpret_cast<GetRange>(fn);
  }();
  unsigned long long b = 0;
  size_t sz = 0;
  if (!get_range || get_range(&b, &sz, reinterpret_cast<unsigned long long>(p)) != 0)
    return false;
  *base = static_cast<uintptr_t>(b);
  *size = sz;
  return true;
}

// Allocations of other processes mapped into this one (mp_ipc_import),
// per importing device, reference counted (mp_ipc_close).
struct IpcMapping {
  int dev;
  std::string handle;
  void *base;
  size_t size;
  size_t refs;
};
std::mutex g_ipc_mu;
std::vector<IpcMapping> g_ipc;

// Is p inside memory mapped from another process?  Such memory may live on
// another GPU whatever the pointer attributes report, so the piece merge
// reads it with LSU loads (valid for peer and local memory alike).
bool is_ipc_mapped(const void *p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  for (const auto &e : g_ipc) {
    const uintptr_t b = reinterpret_cast<uintptr_t>(e.base);
    if (a >= b && a < b + e.size)
      return true;
  }
  return false;
}

template <class KT> bool aligned_keys(const void *p) {
  return (reinterpret_cast<uintptr_t>(p) % alignof(typename KT::T)) == 0;
}

// ---- per-key-type tile shapes --------------------------------------------
// Plain merge: odd VT (conflict-free staging, bulk-store epilogue).
#ifndef MP_MERGE_NT
#define MP_MERGE_NT 256
#endif
// B200 A/B (tools/merge_variants.py, ms): VT4 15 -> 23: config 2 0.672 ->
// 0.666, random u32 2^28+2^28 0.784 -> 0.713; VT8 11 beats 15 on config 3a.
#ifndef MP_MERGE_VT4
#define MP_MERGE_VT4 23
#endif
#ifndef MP_MERGE_VT8
#define MP_MERGE_VT8 11
#endif
// Bare 4-byte integer keys take twice the tile (NT 512): half the K1 split
// searches, same K2 rate.  B200 A/B (200 steps, tools/variants): config 2
// step 0.671 -> 0.662 ms; but u32 + values 0.662 -> 0.741 ms, config 3a
// (u64 + values) 2.05 -> 2.43 ms and config 5 (f32) 6.37 -> 6.48 ms at 512,
// so values, the checksum sink and other key types keep NT 256.
#ifndef MP_MERGE_NT_I4
#define MP_MERGE_NT_I4 512
#endif
template <class KT> struct MergeCfg {
  // the tile the split search (K1, mp_merge_plan) is planned at
  static constexpr int NT =
      (KT::kind == kU32 || KT::kind == kI32) ? MP_MERGE_NT_I4 : MP_MERGE_NT;
  static constexpr int VT = sizeof(typename KT::T) == 4   ? MP_MERGE_VT4
                            : sizeof(typename KT::T) == 8 ? MP_MERGE_VT8
                                                          : 7;
  // the tile K2 runs at for a given payload: values / the register sink
  // use NT 256; a plan at a wider tile is refined (refine_partition_kernel)
  template <bool VALS, bool SINK>
  static constexpr int exec_nt() { return (VALS || SINK) ? MP_MERGE_NT : NT; }
};
// Sort rounds: the tile (TILE outputs) must divide 2 * 2048 (block-sort run
// length) so no tile straddles two run pairs.  TILE is a power of two, but
// the thread shape keeps VT odd (conflict-free smem access, bulk-store
// epilogue) with NT*VT >= TILE; surplus threads own empty diagonals.
template <class KT> struct SortMergeCfg {
  static constexpr int TILE = sizeof(typename KT::T) == 4   ? 4096
                              : sizeof(typename KT::T) == 8 ? 2048
                                                            : 1024;
#ifndef MP_SORT_VT4
#define MP_SORT_VT4 23  // B200 A/B (tools/sort_variants.py): 15 38.1 ms,
#endif                  // 19 39.4, 23 35.9, 31 41.3 for 2^30 u32 keys
  static constexpr int VT = sizeof(typename KT::T) == 4   ? MP_SORT_VT4
                            : sizeof(typename KT::T) == 8 ? 11
                                                          : 7;
  static constexpr int NT = ((TILE + VT - 1) / VT + 31) / 32 * 32;
};
constexpr int kBlockNT = 128;
constexpr int kBlockVT = 16;
constexpr uint64_t kRun = kBlockNT * kBlockVT;  // 2048-key block-sort runs
// bare 32-bit keys: K3w (mp_bsort.cuh)
#ifndef MP_WARP_NT
#define MP_WARP_NT 256
#endif
constexpr int kWarpNT = MP_WARP_NT;
// K3w shape: 16384-key runs, so a 2^30-key sort is 16 rounds = 8 fused round
// pairs with no plain round left over.  B200 A/B (tools/ab_k3w_shape.sh,
// whole 2^30 sort / K3w alone, 1965 MHz): 512 x 16 (8192-key runs, 4 smem
// passes) 27.27 / 7.59 ms; 256 x 32 (8192-key runs, 3 smem passes) 26.68 /
// 7.00 ms; 512 x 32 26.53 / 8.05 ms; 256 x 64 (16384-key runs, 3 smem passes,
// 80 registers, tools/ab_k3w_v64.sh) 26.27 / 8.04 ms with K5e's granule
// copies vs 26.27-26.34 for 512 x 32.  With the FMA-pipe compare-exchanges
// (mp_bsort.cuh) a register-network level costs ~0.4 ms against ~1 ms for a
// shared-memory pass, and 256 x 64 (2048 keys per warp in registers, one pass
// less) wins: 25.58 / 7.33 ms vs 25.78 / 7.54 for 512 x 32.
#ifndef MP_K3W_VT
#define MP_K3W_VT 64
#endif
constexpr int kWarpVT = MP_K3W_VT;
uint64_t warp_run() { return uint64_t(kWarpNT) * kWarpVT; }

constexpr uint32_t kBigTile4 = 8192;  // round tile after K3w (sort_round_tile)
constexpr int kBigTileNT = 384;       // 384 x 23 >= 8192
// K5e (fused two-round pass) thread shape at the 8192-output tile:
// QNT * QVT >= 8192 + 2 * QVT, QVT odd
// B200 A/B (tools/ab_qshape.sh, ab_q16k.sh, whole 2^30 sort): at the
// 8192-output tile 384 x 23 29.49 ms, 288 x 31 29.11, 320 x 27 29.01; at
// the 16384-output tile 640 x 27 28.17-28.32 (K4q + K4r per pass 0.39 ->
// 0.18 ms, K5e 2.07 -> 2.13 ms), 544 x 31 29.28, 576 x 29 28.14, 704 x 25
// 28.54.  Round 2, after the granule copies (tools/ab_qshape2.sh, 2^30
// sort): 640 x 27 26.27, 576 x 29 26.25, 672 x 25 26.52, 704 x 25 28.49 ms.
#ifndef MP_QUAD_NT
#define MP_QUAD_NT 640
#endif
#ifndef MP_QUAD_VT
#define MP_QUAD_VT 27
#endif
constexpr int kQuadNT = MP_QUAD_NT;
constexpr int kQuadVT = MP_QUAD_VT;
// the fused pass's output tile after K3w's runs (a multiple of the round
// tile that divides 4 x 8192)
#ifndef MP_QUAD_TILE
#define MP_QUAD_TILE 16384
#endif
constexpr uint32_t kQuadTile = MP_QUAD_TILE;
static_assert(kQuadNT * kQuadVT >= int(kQuadTile) + 2 * kQuadVT && (kQuadVT & 1),
              "K5e at the fused-pass tile");

template <class K> cudaError_t set_smem(K kernel, uint32_t bytes) {
  if (bytes <= 48 * 1024)
    return cudaSuccess;
  return cudaFuncSetAttribute(kernel,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(bytes));
}

// ---- K1 -------------------------------------------------------------------
template <class KT>
int launch_partition(const void *a, uint64_t na, const void *b, uint64_t nb,
                     uint64_t spacing, uint64_t p, uint64_t count,
                     uint64_t *a_offs, cudaStream_t s,
                     uint64_t *cmp = nullptr) {
  using T = typename KT::T;
  if (count == 0)
    return MP_OK;
  const unsigned blocks = static_cast<unsigned>(cdiv(count, 128));
  partition_kernel<KT><<<blocks, 128, 0, s>>>(
      static_cast<const T *>(a), na, static_cast<const T *>(b), nb, spacing, p,
      count, a_offs, reinterpret_cast<unsigned long long *>(cmp));
  MP_LAUNCHED("partition_kernel");
  return MP_OK;
}

// ---- K1 + K2: plain merge --------------------------------------------------
// Workspace of a plain merge = the tile partition array P[0..tiles].
template <class KT> uint64_t merge_tiles(uint64_t n) {
  constexpr uint64_t NV = MergeCfg<KT>::NT * MergeCfg<KT>::VT;
  return cdiv(n, NV);
}
// + the refined (NT 256) split points when the plan tile is wider
template <class KT> uint64_t merge_ws_bytes(uint64_t n) {
  if (!n)
    return 0;
  constexpr uint64_t NVe = uint64_t(MP_MERGE_NT) * MergeCfg<KT>::VT;
  const uint64_t fine = MergeCfg<KT>::NT == MP_MERGE_NT ? 0 : cdiv(n, NVe) + 1;
  return (merge_tiles<KT>(n) + 1 + fine) * sizeof(uint64_t);
}

// Merges (and sort rounds) of at most this many tiles run as ONE kernel:
// each K2 CTA searches its own split points (SearchMap / RoundSearchMap),
// no K1/K4 launch.  The in-CTA search costs every CTA ~1-2 us of latency,
// which the saved launch outweighs up to a few waves.  B200 A/B
// (tools/small_probe.py, us per call, threshold 592 -> 3072 -> 4096):
// merge 2^23 u32 24.6 -> 16.5, 3*2^23 54.0 -> 50.7; sort 2^23 301 -> 247,
// 2^24 557 -> 510, 2^25 960 -> 962 -> 985 (4096 round tiles: worse);
// always on: sort 2^28 6.97 -> 8.45 ms.  MP_MERGE_FUSE_TILES overrides
// (0 = always K1/K4 + K2).
uint64_t merge_fuse_tiles() {
  static const uint64_t v = [] {
    const char *e = std::getenv("MP_MERGE_FUSE_TILES");
    return e ? static_cast<uint64_t>(std::atoll(e)) : uint64_t(3072);
  }();
  return v;
}
// K4 with a warp per tile boundary up to this many tiles (MP_K4_WARP_TILES):
// B200 sort (tools/small_probe.py), us: 2^25 (4096 round tiles) 961 -> 921,
// but 2^26 (8192) 1776 -> 1862 and 2^27 3454 -> 3805 -- the warp search's
// 32x sectors cost more than its latency saves once K4 has many tiles.
uint64_t k4_warp_tiles() {
  static const uint64_t v = [] {
    const char *e = std::getenv("MP_K4_WARP_TILES");
    return e ? static_cast<uint64_t>(std::atoll(e)) : uint64_t(4096);
  }();
  return v;
}
template <class KT> bool merge_fused(uint64_t n) {
  return cdiv(n, uint64_t(MergeCfg<KT>::NT) * MergeCfg<KT>::VT) <= merge_fuse_tiles();
}

// K1 at tile spacing: P[t] = a_off on diagonal t*NV.  (Nothing to do for a
// fused small merge: merge_exec's CTAs search their own split points.)
template <class KT>
int merge_plan(const void *a, uint64_t na, const void *b, uint64_t nb,
               uint64_t *P, cudaStream_t s) {
  constexpr uint64_t NV = MergeCfg<KT>::NT * MergeCfg<KT>::VT;
  const uint64_t n = na + nb;
  if (n == 0 || merge_fused<KT>(n))
    return MP_OK;
  if (merge_tiles<KT>(n) >= (1ull << 31))
    return fail(MP_ERR_INVALID, "merge too large (%llu elements)",
                (unsigned long long)n);
  return launch_partition<KT>(a, na, b, nb, NV, 0, merge_tiles<KT>(n) + 1, P,
                              s);
}

// K2 over the tiles planned by merge_plan.
template <class KT, bool VALS, bool SINK>
int merge_exec(const void *a, const uint32_t *av, uint64_t na, const void *b,
               const uint32_t *bv, uint64_t nb, void *out, uint32_t *outv,
               unsigned long long *sum, const uint64_t *P, cudaStream_t s) {
  using T = typename KT::T;
  constexpr int NT = MergeCfg<KT>::template exec_nt<VALS, SINK>(), VT = MergeCfg<KT>::VT;
  constexpr uint32_t NV = NT * VT;
  const uint64_t n = na + nb;
  if (n == 0)
    return MP_OK;
  const uint64_t tiles = cdiv(n, NV);
  if (merge_fused<KT>(n)) {
    constexpr uint32_t smem = merge_smem_bytes<KT, VALS, NT, VT>();
    auto kern = merge_tiles_kernel<KT, VALS, NT, VT, SearchMap, SINK>;
    MP_CUDA(set_smem(kern, smem));
    kern<<<static_cast<unsigned>(tiles), NT, smem, s>>>(
        SearchMap{na, n, NV}, static_cast<const T *>(a), av, static_cast<const T *>(b), bv,
        static_cast<T *>(out), outv, sum, 0);
    MP_LAUNCHED("merge_tiles_kernel(search)");
    return MP_OK;
  }
  if constexpr (NT != MergeCfg<KT>::NT) {
    // the plan is at the wider tile: refine it to this tile's split points
    // (bounded searches between neighbouring planned points), stored behind
    // the planned ones in the workspace
    constexpr uint32_t R = MergeCfg<KT>::NT / NT;
    static_assert(MergeCfg<KT>::NT % NT == 0, "plan tile = R exec tiles");
    uint64_t *Pf = const_cast<uint64_t *>(P) + merge_tiles<KT>(n) + 1;
    refine_partition_kernel<KT>
        <<<static_cast<unsigned>(cdiv(tiles + 1, 128)), 128, 0, s>>>(
            static_cast<const T *>(a), na, static_cast<const T *>(b), nb, P, NV, R,
            tiles + 1, Pf);
    MP_LAUNCHED("refine_partition_kernel");
    P = Pf;
  }
  constexpr uint32_t smem = merge_smem_bytes<KT, VALS, NT, VT>();
  auto kern = merge_tiles_kernel<KT, VALS, NT, VT, PlainMap, SINK>;
  MP_CUDA(set_smem(kern, smem));
  kern<<<static_cast<unsigned>(tiles), NT, smem, s>>>(
      PlainMap{P, n, NV}, static_cast<const T *>(a), av, static_cast<const T *>(b), bv,
      static_cast<T *>(out), outv, sum, 0);
  MP_LAUNCHED("merge_tiles_kernel");
  return MP_OK;
}

template <class KT, bool VALS, bool SINK>
int merge_impl(const void *a, const uint32_t *av, uint64_t na, const void *b,
               const uint32_t *bv, uint64_t nb, void *out, uint32_t *outv,
               unsigned long long *sum, cudaStream_t s) {
  using T = typename KT::T;
  // one-shot: plan and merge at the payload's own tile
  constexpr int NT = MergeCfg<KT>::template exec_nt<VALS, SINK>(), VT = MergeCfg<KT>::VT;
  constexpr uint32_t NV = NT * VT;
  const uint64_t n = na + nb;
  if (n == 0)
    return MP_OK;
  const uint64_t tiles = cdiv(n, NV);
  if (tiles >= (1ull << 31))
    return fail(MP_ERR_INVALID, "merge too large (%llu elements)",
                (unsigned long long)n);
  constexpr uint32_t smem = merge_smem_bytes<KT, VALS, NT, VT>();
  if (merge_fused<KT>(n)) {  // a few waves: CTAs search their own splits
    auto kern = merge_tiles_kernel<KT, VALS, NT, VT, SearchMap, SINK>;
    MP_CUDA(set_smem(kern, smem));
    kern<<<static_cast<unsigned>(tiles), NT, smem, s>>>(
        SearchMap{na, n, NV}, static_cast<const T *>(a), av, static_cast<const T *>(b), bv,
        static_cast<T *>(out), outv, sum, 0);
    MP_LAUNCHED("merge_tiles_kernel(search)");
    return MP_OK;
  }
  ScratchGuard P;
  if (int rc = alloc_scratch(P, merge_ws_bytes<KT>(n), s))
    return rc;
  uint64_t *Pp = static_cast<uint64_t *>(P.p);
  partition_kernel<KT><<<static_cast<unsigned>(cdiv(tiles + 1, 128)), 128, 0, s>>>(
      static_cast<const T *>(a), na, static_cast<const T *>(b), nb, NV, 0, tiles + 1, Pp,
      nullptr);
  MP_LAUNCHED("partition_kernel");
  auto kern = merge_tiles_kernel<KT, VALS, NT, VT, PlainMap, SINK>;
  MP_CUDA(set_smem(kern, smem));
  kern<<<static_cast<unsigned>(tiles), NT, smem, s>>>(
      PlainMap{Pp, n, NV}, static_cast<const T *>(a), av, static_cast<const T *>(b), bv,
      static_cast<T *>(out), outv, sum, 0);
  MP_LAUNCHED("merge_tiles_kernel");
  return MP_OK;
}

// ---- K3 + (K4 + K2) x rounds: bottom-up merge sort ---------------------------
struct SortLayout {
  uint64_t keys_off, vals_off, part_off, quad_off, total;
};
// grid spacing of the fused two-round pass (mp_quad.cuh): the bare block
// sort's run, so G divides every pair width 2w

template <class KT> SortLayout sort_layout(bool vals, uint64_t n) {
  using T = typename KT::T;
  constexpr uint64_t NV = SortMergeCfg<KT>::TILE;
  auto up = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  SortLayout L;
  L.keys_off = 0;
  L.vals_off = up(n * sizeof(T));
  L.part_off = L.vals_off + (vals ? up(n * 4) : 0);
  L.quad_off = L.part_off + up((cdiv(n, NV) + 1) * sizeof(uint64_t));
  L.total = L.quad_off +
            (!vals && sizeof(T) == 4 ? up((2 * cdiv(n, 4096) + 32) * sizeof(QuadPt)) : 0);
  return L;
}

// Block sort of bare 32-bit keys: K3w (mp_bsort.cuh, 8192-key runs) by
// default; MP_BLOCK_SORT=merge selects the stable K3 (2048-key runs) for
// them too (tests the generic path on bare keys).  Measured-slower
// alternatives (K3b 4352-key runs: 33.1 vs 31.6 ms per 2^30 sort; K3t:
// 8.44 vs 8.26 ms per block pass; an LSD radix block sort with match.any
// ranking: 30 ms for the block pass alone) are in tools/variants/.
bool block_sort_generic() {
  static const bool b = [] {
    const char *v = std::getenv("MP_BLOCK_SORT");
    return v && std::strcmp(v, "merge") == 0;
  }();
  return b;
}

// Run length the block sort leaves and the round tile (mp_sort's schedule).
template <class KT, bool VALS> uint64_t sort_run0() {
  constexpr bool bare4 = !VALS && sizeof(typename KT::T) == 4 && KT::kind != kElement;
  return bare4 && !block_sort_generic() ? warp_run() : kRun;
}
// Fused two-round passes (mp_quad.cuh) for bare 32-bit sorts whose rounds
// are too large for the in-kernel split search: default on, MP_SORT_QUAD=0
// turns them off (=1 forces them at every size).
int sort_quad_env() {
  static const int v = [] {
    const char *e = std::getenv("MP_SORT_QUAD");
    return !e ? 2 : std::strcmp(e, "0") == 0 ? 0 : 1;
  }();
  return v;
}
// Round tile after K3w's 8192-key runs: kBigTile4 (8192 = 384 threads x 23
// outputs: half the K4 split searches of 4096-output tiles) unless
// MP_SORT_TILE=4096.
bool sort_big_tile_env() {
  static const bool b = [] {
    const char *e = std::getenv("MP_SORT_TILE");
    return !(e && std::atoi(e) == 4096);
  }();
  return b;
}
template <class KT, bool VALS> uint32_t sort_round_tile() {
  const uint64_t r0 = sort_run0<KT, VALS>();
  if (sizeof(typename KT::T) == 4 && !VALS && KT::kind != kElement && r0 % kBigTile4 == 0 &&
      sort_big_tile_env())
    return kBigTile4;
  return SortMergeCfg<KT>::TILE;
}

// Plain bottom-up rounds over sorted runs of width w0 held in `src`
// (sort.hpp:71-128): per round K4 (pair-local split points at tile NV) and
// K2 over RoundMap, ping-pong src <-> dst.  *res / *resv receive the buffer
// holding the result.
template <class KT, bool VALS, int NT = SortMergeCfg<KT>::NT, int VT = SortMergeCfg<KT>::VT>
int sort_rounds_from(typename KT::T *src, uint32_t *srcv, typename KT::T *dst,
                     uint32_t *dstv, uint64_t n, uint64_t w0, uint32_t NV,
                     uint64_t *P, cudaStream_t s, typename KT::T **res,
                     uint32_t **resv) {
  using T = typename KT::T;
  if constexpr (sizeof(T) == 4 && !VALS && NT == SortMergeCfg<KT>::NT) {
    if (NV > static_cast<uint32_t>(NT * VT))  // kBigTile4 rounds after K3w
      return sort_rounds_from<KT, VALS, kBigTileNT, VT>(src, srcv, dst, dstv, n, w0, NV, P, s,
                                                        res, resv);
  }
  const uint64_t tiles = cdiv(n, NV);
  constexpr uint32_t smem = merge_smem_bytes<KT, VALS, NT, VT>();
  auto kern = merge_tiles_kernel<KT, VALS, NT, VT, RoundMap, false>;
  MP_CUDA(set_smem(kern, smem));
  uint32_t tshift = static_cast<uint32_t>(__builtin_ctzll(2 * w0 / NV));  // 2w = NV << tshift
  for (uint64_t w = w0; w < n; w *= 2, ++tshift) {
    if (tiles <= merge_fuse_tiles()) {  // a few waves: CTAs search their own splits
      auto kfs = merge_tiles_kernel<KT, VALS, NT, VT, RoundSearchMap, false>;
      MP_CUDA(set_smem(kfs, smem));
      kfs<<<static_cast<unsigned>(tiles), NT, smem, s>>>(
          RoundSearchMap{n, w, NV, tshift}, src, srcv, src, srcv, dst, dstv, nullptr, 0);
      MP_LAUNCHED("merge_tiles_kernel(round, search)");
    } else {
      // K4: pair-local split points at every tile start, then K2
      if (tiles <= k4_warp_tiles()) {
        round_partition_warp_kernel<KT>
            <<<static_cast<unsigned>(cdiv(tiles * 32, 256)), 256, 0, s>>>(
                src, n, w, tshift, NV, tiles, P);
        MP_LAUNCHED("round_partition_warp_kernel");
      } else {
        round_partition_kernel<KT><<<static_cast<unsigned>(cdiv(tiles, 128)), 128, 0, s>>>(
            src, n, w, tshift, NV, tiles, P);
        MP_LAUNCHED("round_partition_kernel");
      }
      kern<<<static_cast<unsigned>(tiles), NT, smem, s>>>(
          RoundMap{P, n, w, NV, tshift}, src, srcv, src, srcv, dst, dstv, nullptr, 0);
      MP_LAUNCHED("merge_tiles_kernel(round)");
    }
    std::swap(src, dst);
    std::swap(srcv, dstv);
  }
  if (res)
    *res = src;
  if (resv)
    *resv = srcv;
  return MP_OK;
}

template <class KT, bool VALS>
int sort_impl(const void *in_, const uint32_t *inv, void *keys_,
              uint32_t *vals, uint64_t n, void *scratch,
              uint64_t scratch_bytes, cudaStream_t s) {
  using T = typename KT::T;
  T *keys = static_cast<T *>(keys_);
  const T *in = static_cast<const T *>(in_);
  if (n <= 1) {
    if (n == 1 && in != keys)
      MP_CUDA(cudaMemcpyAsync(keys, in, sizeof(T), cudaMemcpyDeviceToDevice, s));
    if (VALS && n == 1 && inv != vals)
      MP_CUDA(cudaMemcpyAsync(vals, inv, 4, cudaMemcpyDeviceToDevice, s));
    return MP_OK;
  }
  const SortLayout L = sort_layout<KT>(VALS, n);
  ScratchGuard own;
  char *ws = static_cast<char *>(scratch);
  if (!ws) {
    if (int rc = alloc_scratch(own, L.total, s))
      return rc;
    ws = static_cast<char *>(own.p);
  } else if (scratch_bytes < L.total) {
    return fail(MP_ERR_INVALID, "scratch too small: %llu < %llu bytes",
                (unsigned long long)scratch_bytes,
                (unsigned long long)L.total);
  }
  T *aux = reinterpret_cast<T *>(ws + L.keys_off);
  uint32_t *auxv = VALS ? reinterpret_cast<uint32_t *>(ws + L.vals_off) : nullptr;
  uint64_t *P = reinterpret_cast<uint64_t *>(ws + L.part_off);

  constexpr bool kBare4 = !VALS && sizeof(T) == 4 && KT::kind != kElement;
  const bool use_warp = kBare4 && !block_sort_generic();  // K3w runs
  const uint64_t run0 = use_warp ? warp_run() : kRun;
  int rounds = 0;
  for (uint64_t w = run0; w < n; w *= 2)
    ++rounds;
  // Fused round pairs: one HBM pass per two rounds (mp_quad.cuh).  B200,
  // 2^30 u32, per pass at the 16384-output tile: K4q 0.05 + K4r 0.13 + K5e
  // 2.1 ms vs 2 x (1.23 + 0.06) ms for two plain rounds; with half the HBM
  // traffic the sort also stays under the power cap.  Small sorts keep the
  // plain rounds (their in-kernel split search is cheaper than K4q + K4r).
  const int quad_mode = kBare4 ? sort_quad_env() : 0;
  const bool use_quad =
      quad_mode == 1 ||
      (quad_mode == 2 && cdiv(n, uint64_t(sort_round_tile<KT, VALS>())) > merge_fuse_tiles());
  const int quad_passes = use_quad ? rounds / 2 : 0;
  const int passes = rounds - quad_passes;  // ping-pong swaps after the block sort
  // Block sort lands where an even/odd number of ping-pong passes ends in
  // `keys` (the result always lands back in the caller's buffer).
  const bool in_place = (passes % 2) == 0;
  T *src = in_place ? keys : aux;
  uint32_t *srcv = in_place ? vals : auxv;
  T *dst = in_place ? aux : keys;
  uint32_t *dstv = in_place ? auxv : vals;

  if (use_warp) {
    if constexpr (kBare4) {
      const bool al = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
      constexpr uint64_t run = uint64_t(kWarpNT) * kWarpVT;
      const uint64_t whole = al ? n / run : 0, blocks = cdiv(n, run);
      constexpr uint32_t smem = warp_sort_smem_bytes<kWarpNT, kWarpVT>();
      if (whole) {
        auto kern = block_sort_warp_kernel<KT, kWarpNT, true, kWarpVT>;
        MP_CUDA(set_smem(kern, smem));
        kern<<<static_cast<unsigned>(whole), kWarpNT, smem, s>>>(in, src, n, 0, 1u);
        MP_LAUNCHED("block_sort_warp_kernel");
      }
      if (blocks > whole) {
        auto kern = block_sort_warp_kernel<KT, kWarpNT, false, kWarpVT>;
        MP_CUDA(set_smem(kern, smem));
        kern<<<static_cast<unsigned>(blocks - whole), kWarpNT, smem, s>>>(in, src, n, whole, 1u);
        MP_LAUNCHED("block_sort_warp_kernel(tail)");
      }
    }
  } else {
    constexpr uint32_t smem = block_sort_smem_bytes<KT, VALS, kBlockNT, kBlockVT>();
    auto kern = block_sort_kernel<KT, VALS, kBlockNT, kBlockVT>;
    MP_CUDA(set_smem(kern, smem));
    kern<<<static_cast<unsigned>(cdiv(n, kRun)), kBlockNT, smem, s>>>(
        in, inv, src, srcv, n);
    MP_LAUNCHED("block_sort_kernel");
  }

  constexpr int NT = SortMergeCfg<KT>::NT, VT = SortMergeCfg<KT>::VT;
  // round tile: it divides every pair width with a power-of-two ratio
  static_assert(NT * VT >= int(SortMergeCfg<KT>::TILE) && (2 * kRun) % SortMergeCfg<KT>::TILE == 0,
                "round tile shape");
  const uint32_t NV = sort_round_tile<KT, VALS>();
  uint64_t w = run0;
  if constexpr (kBare4) {
    // fused round pairs (mp_quad.cuh v2): K4q crossings at grid G = NV,
    // K4r exact 4-way splits at every NV-output tile, K5e tile merges
    for (int fused_left = quad_passes; fused_left > 0 && w < n; --fused_left, w *= 4) {
      QuadPt *QP = reinterpret_cast<QuadPt *>(ws + L.quad_off);
      // the fused pass's tile QT (and crossing grid) may be wider than the
      // plain rounds' tile: kQuadTile after K3w's runs
      const uint32_t QT = NV == kBigTile4 ? kQuadTile : NV;
      const uint32_t G = QT;
      const uint32_t lshift = static_cast<uint32_t>(__builtin_ctzll(4 * w / G));
      const uint64_t full = n / (4 * w);
      uint64_t lines = full << lshift;
      if (full * 4 * w < n) {  // short last group
        const uint64_t S = full * 4 * w;
        uint64_t l[4];
        for (int r = 0; r < 4; ++r) {
          const uint64_t st = S + r * w;
          l[r] = st < n ? std::min<uint64_t>(w, n - st) : 0;
        }
        lines += cdiv(l[0] + l[1], G) + cdiv(l[2] + l[3], G);
      }
      const uint64_t qtiles = cdiv(n, QT);
      QuadPt *QQ = QP + cdiv(n, G) + 8;
      auto launch = [&](auto g_tag) -> int {
        constexpr uint32_t GG = decltype(g_tag)::value;
        quad_partition_kernel<KT, GG><<<static_cast<unsigned>(cdiv(lines, 128)), 128, 0, s>>>(
            src, n, w, lshift, lines, QP);
        MP_LAUNCHED("quad_partition_kernel");
        quad_refine_kernel<KT, GG><<<static_cast<unsigned>(cdiv(qtiles, 128)), 128, 0, s>>>(
            src, n, w, lshift, QT, qtiles, QP, QQ);
        MP_LAUNCHED("quad_refine_kernel");
        return MP_OK;
      };
      int rc = QT == kQuadTile ? launch(std::integral_constant<uint32_t, kQuadTile>{})
                               : launch(std::integral_constant<uint32_t, 4096u>{});
      if (rc)
        return rc;
      const uint32_t lg4w = ((4 * w) & (4 * w - 1)) == 0
                                ? static_cast<uint32_t>(__builtin_ctzll(4 * w))
                                : ~0u;
      auto tiles_k5 = [&](auto nt_tag) -> int {
        constexpr int QNT = decltype(nt_tag)::value;
        constexpr int QVT = QNT == kQuadNT ? kQuadVT : VT;
        static_assert(QNT * QVT >= 4096 + 2 * QVT, "K5e: a tile's two inner merges fit the CTA");
        constexpr uint32_t qsmem = quad_smem_bytes<KT, QNT, QVT>();
        auto qkern = quad_tile_kernel<KT, QNT, QVT>;
        MP_CUDA(set_smem(qkern, qsmem));
        qkern<<<static_cast<unsigned>(qtiles), QNT, qsmem, s>>>(src, dst, n, w, lg4w, QT, QQ);
        MP_LAUNCHED("quad_tile_kernel");
        return MP_OK;
      };
      rc = QT == kQuadTile ? tiles_k5(std::integral_constant<int, kQuadNT>{})
                           : tiles_k5(std::integral_constant<int, NT>{});
      if (rc)
        return rc;
      std::swap(src, dst);
    }
  }
  return sort_rounds_from<KT, VALS>(src, srcv, dst, dstv, n, w, NV, P, s, nullptr, nullptr);
}

// ---- generators -------------------------------------------------------------
__global__ void generate_kernel(int kind, uint64_t seed, uint64_t first,
                                uint64_t n, void *out) {
  const uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (k >= n)
    return;
  const uint64_t x = mix64_dev(seed + (first + k) * 0x9E3779B97F4A7C15ULL);
  switch (kind) {
  case 0:
    static_cast<uint32_t *>(out)[k] = static_cast<uint32_t>(x >> 32);
    break;
  case 1:
    static_cast<int32_t *>(out)[k] = static_cast<int32_t>(x >> 54);
    break;
  case 2:
    static_cast<unsigned long long *>(out)[k] = x;
    break;
  case 3:
    static_cast<unsigned long long *>(out)[k] = x >> 24;
    break;
  case 4:
    static_cast<unsigned long long *>(out)[k] =
        (1ull << 40) + __umul64hi(x, ~0ull - (1ull << 40) + 1ull);
    break;
  case 5: {  // Normal(0,1), Box-Muller cosine branch
    const uint64_t i = first + k;
    const uint64_t x0 = mix64_dev(seed + (2 * i) * 0x9E3779B97F4A7C15ULL);
    const uint64_t x1 = mix64_dev(seed + (2 * i + 1) * 0x9E3779B97F4A7C15ULL);
    const double u1 = static_cast<double>((x0 >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(x1 >> 11) * 0x1.0p-53;
    static_cast<float *>(out)[k] =
        static_cast<float>(sqrt(-2.0 * log(u1)) * cospi(2.0 * u2));
    break;
  }
  case 6: {  // Exp(1)
    const double u = static_cast<double>((x >> 11) + 1) * 0x1.0p-53;
    static_cast<float *>(out)[k] = static_cast<float>(-log(u));
    break;
  }
  }
}

// ---- dispatch --------------------------------------------------------------
template <template <class> class F, class... Args>
int dispatch(int kt, Args &&...args) {
  switch (kt) {
  case kU32:
    return F<KeyU32>::run(args...);
  case kI32:
    return F<KeyI32>::run(args...);
  case kF32:
    return F<KeyF32>::run(args...);
  case kU64:
    return F<KeyU64>::run(args...);
  case kI64:
    return F<KeyI64>::run(args...);
  case kElement:
    return F<KeyElement>::run(args...);
  default:
    return fail(MP_ERR_UNSUPPORTED, "unknown key type %d", kt);
  }
}

template <class KT> struct PartitionOp {
  static int run(const void *a, uint64_t na, const void *b, uint64_t nb,
                 uint64_t p, uint64_t *a_offs, uint64_t *cmp, cudaStream_t s) {
    if (!aligned_keys<KT>(a) || !aligned_keys<KT>(b))
      return fail(MP_ERR_INVALID, "misaligned key pointer");
    return launch_partition<KT>(a, na, b, nb, 0, p, p + 1, a_offs, s, cmp);
  }
};

template <class KT> struct DiagonalsOp {
  static int run(const void *a, uint64_t na, const void *b, uint64_t nb,
                 const uint64_t *diags, uint64_t count, uint64_t *a_offs,
                 uint64_t *cmp, cudaStream_t s) {
    using T = typename KT::T;
    if (count == 0)
      return MP_OK;
    diagonals_kernel<KT><<<static_cast<unsigned>(cdiv(count, 128)), 128, 0, s>>>(
        static_cast<const T *>(a), na, static_cast<const T *>(b), nb, diags,
        count, a_offs, reinterpret_cast<unsigned long long *>(cmp));
    MP_LAUNCHED("diagonals_kernel");
    return MP_OK;
  }
};

// phase 0: plan + execute with a pool workspace; 1: plan into ws;
// 2: execute with a planned ws.
template <class KT> struct MergeOp {
  static int run(const void *a, const uint32_t *av, uint64_t na, const void *b,
                 const uint32_t *bv, uint64_t nb, void *out, uint32_t *outv,
                 int phase, uint64_t *ws, cudaStream_t s) {
    if (!aligned_keys<KT>(a) || !aligned_keys<KT>(b) ||
        (phase != 1 && !aligned_keys<KT>(out)))
      return fail(MP_ERR_INVALID, "misaligned key pointer");
    if (phase == 1)
      return merge_plan<KT>(a, na, b, nb, ws, s);
    const bool vals = av || bv || outv;
    if (vals) {
      if (KT::kind == kElement)
        return fail(MP_ERR_UNSUPPORTED, "ELEMENT keys carry their own tag");
      if (!outv || (na && !av) || (nb && !bv))
        return fail(MP_ERR_INVALID, "values must be given for A, B and out");
      if (phase == 2)
        return merge_exec<KT, true, false>(a, av, na, b, bv, nb, out, outv,
                                           nullptr, ws, s);
      return merge_impl<KT, true, false>(a, av, na, b, bv, nb, out, outv,
                                         nullptr, s);
    }
    if (phase == 2)
      return merge_exec<KT, false, false>(a, nullptr, na, b, nullptr, nb, out,
                                          nullptr, nullptr, ws, s);
    return merge_impl<KT, false, false>(a, nullptr, na, b, nullptr, nb, out,
                                        nullptr, nullptr, s);
  }
};

template <class KT> struct MergeWsOp {
  static int run(uint64_t n, uint64_t *out) {
    *out = merge_ws_bytes<KT>(n);
    return MP_OK;
  }
};

template <class KT> struct ChecksumOp {
  static int run(const void *a, uint64_t na, const void *b, uint64_t nb,
                 uint64_t *sum, cudaStream_t s) {
    if (!aligned_keys<KT>(a) || !aligned_keys<KT>(b))
      return fail(MP_ERR_INVALID, "misaligned key pointer");
    MP_CUDA(cudaMemsetAsync(sum, 0, sizeof(uint64_t), s));
    return merge_impl<KT, false, true>(
        a, nullptr, na, b, nullptr, nb, nullptr, nullptr,
        reinterpret_cast<unsigned long long *>(sum), s);
  }
};

template <class KT> struct SortOp {
  static int run(const void *in, const uint32_t *inv, void *keys,
                 uint32_t *vals, uint64_t n, void *scratch,
                 uint64_t scratch_bytes, cudaStream_t s) {
    if (!aligned_keys<KT>(keys) || !aligned_keys<KT>(in))
      return fail(MP_ERR_INVALID, "misaligned key pointer");
    if (vals || inv) {
      if (KT::kind == kElement)
        return fail(MP_ERR_UNSUPPORTED, "ELEMENT keys carry their own tag");
      if (!vals || !inv)
        return fail(MP_ERR_INVALID, "values must be given for input and output");
      return sort_impl<KT, true>(in, inv, keys, vals, n, scratch,
                                 scratch_bytes, s);
    }
    return sort_impl<KT, false>(in, nullptr, keys, nullptr, n, scratch,
                                scratch_bytes, s);
  }
};

// Segmented-merge schedule on the device: window starts (K1 at diagonals
// k*L) and the reference's exact comparison counters.
template <class KT> struct SegmentOp {
  static int run(const void *a, uint64_t na, const void *b, uint64_t nb,
                 uint64_t p, uint64_t L, uint64_t *start_a, uint64_t *plan_cmp,
                 uint64_t *merge_cmp, uint64_t *scratch_diags,
                 cudaStream_t s) {
    using T = typename KT::T;
    const uint64_t n = na + nb;
    const uint64_t iters = cdiv(n, L);
    if (iters == 0)
      return MP_OK;
    // window starts = diagonal search at k*L (k = 0..iters-1)
    if (int rc = launch_partition<KT>(a, na, b, nb, L, 0, iters, start_a, s))
      return rc;
    (void)scratch_diags;
    const uint64_t p_eff = p < L ? p : L;
    if (plan_cmp || merge_cmp) {
      ScratchGuard g;
      unsigned long long *pc = reinterpret_cast<unsigned long long *>(plan_cmp);
      unsigned long long *mc = reinterpret_cast<unsigned long long *>(merge_cmp);
      if (!pc || !mc) {
        if (int rc = alloc_scratch(g, 16, s))
          return rc;
        if (!pc)
          pc = static_cast<unsigned long long *>(g.p);
        if (!mc)
          mc = static_cast<unsigned long long *>(g.p) + 1;
      }
      const uint64_t threads = iters * (p_eff + 1);
      segment_stats_kernel<KT>
          <<<static_cast<unsigned>(cdiv(threads, 128)), 128, 0, s>>>(
              static_cast<const T *>(a), na, static_cast<const T *>(b), nb, L,
              p_eff, iters, start_a, pc, mc);
      MP_LAUNCHED("segment_stats_kernel");
    }
    return MP_OK;
  }
};

// Merge of piece-concatenated sequences (mp_pieces.cuh): tile split points
// searched over the virtual index spaces, then one CTA per tile stages its
// windows from the (local or peer-mapped) pieces.  Two launches on the
// caller's stream, no host synchronisation.
// Is p memory of another device than `dev` (a peer mapping)?
bool is_peer(const void *p, int dev) {
  if (!p)
    return false;
  if (is_ipc_mapped(p))
    return true;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice && at.device != dev;
}
// MP_PEER_LSU=1: use the LSU loader for every piece window (tests the peer
// path on a one-GPU box)
bool peer_lsu_forced() {
  static const bool f = [] {
    const char *e = std::getenv("MP_PEER_LSU");
    return e && std::strcmp(e, "1") == 0;
  }();
  return f;
}

template <class KT> constexpr int pieces_vt() { return MergeCfg<KT>::VT; }
constexpr int kPiecesNT = MP_MERGE_NT;

template <class KT> struct PiecesOp {
  static int fill(VPieces &V, const mp_piece *p, int np, bool vals, int dev,
                  const char *which) {
    V.n = np;
    V.peer = 0;
    V.start[0] = 0;
    for (int k = 0; k < np; ++k) {
      V.ptr[k] = p[k].keys;
      V.vptr[k] = p[k].vals;
      V.start[k + 1] = V.start[k] + p[k].len;
      if (p[k].len && (!p[k].keys || !aligned_keys<KT>(p[k].keys) || (vals && !p[k].vals)))
        return fail(MP_ERR_INVALID, "merge_pieces: bad %s piece %d", which, k);
      if (p[k].len && (is_peer(p[k].keys, dev) || (vals && is_peer(p[k].vals, dev))))
        V.peer |= 1u << k;
    }
    return MP_OK;
  }

  static int run(const mp_piece *pa, int npa, const mp_piece *pb, int npb,
                 uint64_t o0, uint64_t o1, void *out_, uint32_t *outv,
                 cudaStream_t s) {
    using T = typename KT::T;
    if (npa < 1 || npb < 1 || npa > kMaxPieces || npb > kMaxPieces)
      return fail(MP_ERR_INVALID, "merge_pieces: 1..%d pieces per input", kMaxPieces);
    const bool vals = outv != nullptr;
    if (KT::kind == kElement && vals)
      return fail(MP_ERR_UNSUPPORTED, "ELEMENT keys carry their own tag");
    int dev = 0;
    MP_CUDA(cudaGetDevice(&dev));
    VPieces A{}, B{};
    if (int rc = fill(A, pa, npa, vals, dev, "A"))
      return rc;
    if (int rc = fill(B, pb, npb, vals, dev, "B"))
      return rc;
    const uint64_t na = A.start[npa], nb = B.start[npb];
    if (o0 > o1 || o1 > na + nb)
      return fail(MP_ERR_INVALID, "merge_pieces: output range out of bounds");
    if (o0 == o1)
      return MP_OK;
    if (!out_ || (reinterpret_cast<uintptr_t>(out_) % alignof(T)))
      return fail(MP_ERR_INVALID, "merge_pieces: bad output pointer");
    constexpr int NT = kPiecesNT, VT = pieces_vt<KT>();
    constexpr uint32_t NV = NT * VT;
    const uint64_t tiles = cdiv(o1 - o0, NV);
    if (tiles >= (1ull << 31))
      return fail(MP_ERR_INVALID, "merge_pieces: range too large");
    ScratchGuard g;
    if (int rc = alloc_scratch(g, (tiles + 1) * 8, s))
      return rc;
    uint64_t *P = static_cast<uint64_t *>(g.p);
    pieces_partition_kernel<KT><<<static_cast<unsigned>(cdiv(tiles + 1, 128)), 128, 0, s>>>(
        A, B, o0, o1, NV, tiles + 1, P);
    MP_LAUNCHED("pieces_partition_kernel");
    const int lsu = peer_lsu_forced() ? 1 : 0;
    if (vals) {
      constexpr uint32_t smem = merge_smem_bytes<KT, true, NT, VT>();
      auto kern = pieces_tiles_kernel<KT, true, NT, VT>;
      MP_CUDA(set_smem(kern, smem));
      kern<<<static_cast<unsigned>(tiles), NT, smem, s>>>(A, B, P, o0, o1,
                                                         static_cast<T *>(out_), outv, lsu);
    } else {
      constexpr uint32_t smem = merge_smem_bytes<KT, false, NT, VT>();
      auto kern = pieces_tiles_kernel<KT, false, NT, VT>;
      MP_CUDA(set_smem(kern, smem));
      kern<<<static_cast<unsigned>(tiles), NT, smem, s>>>(A, B, P, o0, o1,
                                                         static_cast<T *>(out_), nullptr, lsu);
    }
    MP_LAUNCHED("pieces_tiles_kernel");
    return MP_OK;
  }
};

}  // namespace
#include "mp_multi.cuh"
namespace {

template <class KT> struct PiecesDiagOp {
  static int run(const mp_piece *pa, int npa, const mp_piece *pb, int npb,
                 const uint64_t *diags, uint64_t count, uint64_t *a_offs, cudaStream_t s) {
    if (npa < 1 || npb < 1 || npa > kMaxPieces || npb > kMaxPieces)
      return fail(MP_ERR_INVALID, "pieces_partition: 1..%d pieces per input", kMaxPieces);
    if (count == 0)
      return MP_OK;
    if (!diags || !a_offs)
      return fail(MP_ERR_INVALID, "pieces_partition: NULL array");
    int dev = 0;
    MP_CUDA(cudaGetDevice(&dev));
    VPieces A{}, B{};
    if (int rc = PiecesOp<KT>::fill(A, pa, npa, false, dev, "A"))
      return rc;
    if (int rc = PiecesOp<KT>::fill(B, pb, npb, false, dev, "B"))
      return rc;
    pieces_diagonals_kernel<KT><<<static_cast<unsigned>(cdiv(count, 128)), 128, 0, s>>>(
        A, B, diags, count, a_offs);
    MP_LAUNCHED("pieces_diagonals_kernel");
    return MP_OK;
  }
};

template <class KT> struct ScratchOp {
  static int run(bool vals, uint64_t n, uint64_t *out) {
    *out = n <= 1 ? 0 : sort_layout<KT>(vals, n).total;
    return MP_OK;
  }
};

uint64_t key_size(int kt) {
  switch (kt) {
  case kU32:
  case kI32:
  case kF32:
    return 4;
  case kU64:
  case kI64:
    return 8;
  case kElement:
    return 16;
  default:
    return 0;
  }
}

// Host staging: one cached non-blocking stream per device.
cudaStream_t host_stream(int device) {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64)
    return nullptr;
  if (!streams[device])
    cudaStreamCreateWithFlags(&streams[device], cudaStreamNonBlocking);
  return streams[device];
}


// ---------------------------------------------------------------------------
// Pageable host spans.  The drop-in's natural callers hand over std::vector
// memory, which the DMA engines cannot read: the driver then stages it at
// ~11 GB/s.  Instead, the host pipelines below stage pageable chunks
// through pinned buffers with a pool of host threads (memcpy at the host's
// memory bandwidth, ~70-80 GB/s on the B200 box, tools/host_copy_probe.py)
// while the copy engines and the SMs work on neighbouring chunks.
// ---------------------------------------------------------------------------
bool is_pageable(const void *p) {
  if (!p)
    return false;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeUnregistered;
}

// Blocking parallel memcpy over persistent worker threads.
// Host copy with non-temporal stores (SSE2, 64 bytes per iteration): a
// staging copy's destination is read next by a DMA engine (pinned slot) or
// not at all (the caller's output), so write-allocating it in the cache only
// adds a read-for-ownership of every destination line to a copy that is
// bound by host DRAM bandwidth.  glibc's memcpy switches to such stores only
// above ~3/4 of the shared cache, far more than a pool part (1-4 MiB).
// MP_HOST_COPY_NT=0 selects plain memcpy.
#if defined(__x86_64__)
#include <emmintrin.h>
inline void stream_copy(char *dst, const char *src, size_t n) {
  size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
  if (head > n)
    head = n;
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  for (; n >= 64; n -= 64, dst += 64, src += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + 48));
    _mm_stream_si128(reinterpret_cast<__m128i *>(dst), a);
    _mm_stream_si128(reinterpret_cast<__m128i *>(dst + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i *>(dst + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i *>(dst + 48), d);
  }
  _mm_sfence();
  std::memcpy(dst, src, n);
}
#else
inline void stream_copy(char *dst, const char *src, size_t n) { std::memcpy(dst, src, n); }
#endif
inline bool host_copy_nt() {
  static const bool v = [] {
    const char *e = std::getenv("MP_HOST_COPY_NT");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  return v;
}

class CopyPool {
 public:
  static CopyPool &get() {
    static CopyPool pool;
    return pool;
  }
  // copy every (dst, src, bytes) job, each split into pieces over the threads
  void copy(const std::vector<std::tuple<void *, const void *, size_t>> &jobs) {
    std::lock_guard<std::mutex> call(call_mu_);
    size_t total = 0;
    for (const auto &j : jobs)
      total += std::get<2>(j);
    if (!total)
      return;
    // pieces of >= 1 MiB, at most one per thread and job
    std::vector<Part> parts;
    for (const auto &j : jobs) {
      const size_t bytes = std::get<2>(j);
      if (!bytes)
        continue;
      const size_t k = std::max<size_t>(
          1, std::min<size_t>(nthreads_ + 1, bytes >> 20));
      for (size_t q = 0; q < k; ++q) {
        const size_t lo = q * bytes / k, hi = (q + 1) * bytes / k;
        parts.push_back({static_cast<char *>(std::get<0>(j)) + lo,
                         static_cast<const char *>(std::get<1>(j)) + lo, hi - lo});
      }
    }
    {
      // the part list changes only while no worker is inside work()
      std::unique_lock<std::mutex> lk(mu_);
      idle_cv_.wait(lk, [&] { return active_ == 0; });
      parts_.swap(parts);
      next_.store(0);
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == parts_.size(); });
  }

 private:
  struct Part {
    char *dst;
    const char *src;
    size_t bytes;
  };
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    nthreads_ = std::min<unsigned>(hw > 1 ? hw - 1 : 1, 15);
    for (unsigned t = 0; t < nthreads_; ++t)
      threads_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto &t : threads_)
      t.join();
  }
  void work() {
    size_t finished = 0;
    for (size_t i = next_.fetch_add(1); i < parts_.size(); i = next_.fetch_add(1)) {
      if (host_copy_nt())
        stream_copy(parts_[i].dst, parts_[i].src, parts_[i].bytes);
      else
        std::memcpy(parts_[i].dst, parts_[i].src, parts_[i].bytes);
      ++finished;
    }
    if (finished) {
      std::lock_guard<std::mutex> lk(mu_);
      done_ += finished;
      if (done_ == parts_.size())
        done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_)
          return;
        ++active_;
      }
      work();
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--active_ == 0)
          idle_cv_.notify_all();
      }
    }
  }
  unsigned nthreads_ = 1;
  std::vector<std::thread> threads_;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_, idle_cv_;
  std::vector<Part> parts_;
  unsigned active_ = 0;
  std::atomic<size_t> next_{0};
  size_t done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// ---------------------------------------------------------------------------
// Host-buffer merge, pipelined over PCIe.
//
// The output is cut into chunks of Q elements at host-side Merge Path splits
// (the same diagonal search, run on the host arrays: Theorem 14 makes every
// chunk an independent merge).  Chunk k flows through a ring of kSlots
// device slots on three streams:  H2D (copy engine 1) -> K1+K2 (SMs) ->
// D2H (copy engine 2), so the inbound copy of chunk k+1, the merge of chunk
// k and the outbound copy of chunk k-1 overlap.  The bound is
// max(H2D bytes, D2H bytes) / PCIe bandwidth instead of their sum.
// ---------------------------------------------------------------------------
constexpr int kSlots = 4;
constexpr uint64_t kDrainLag = 2;  // pageable outputs: chunks in flight before a drain
static_assert(kSlots > int(kDrainLag), "a drained slot is free before its next D2H");

struct HostPipe {
  std::mutex mu;  // one host call per device at a time
  bool init = false;
  cudaStream_t h2d = nullptr, cmp = nullptr, d2h = nullptr;
  cudaEvent_t ev_h2d[kSlots] = {}, ev_cmp[kSlots] = {}, ev_d2h[kSlots] = {};
  void *buf = nullptr;
  size_t buf_bytes = 0;
  // pinned host staging for pageable callers: kSlots slots in and out
  void *pin = nullptr;
  size_t pin_bytes = 0;

  int setup() {
    if (init)
      return MP_OK;
    MP_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    MP_CUDA(cudaStreamCreateWithFlags(&cmp, cudaStreamNonBlocking));
    MP_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    for (int i = 0; i < kSlots; ++i) {
      MP_CUDA(cudaEventCreateWithFlags(&ev_h2d[i], cudaEventDisableTiming));
      MP_CUDA(cudaEventCreateWithFlags(&ev_cmp[i], cudaEventDisableTiming));
      MP_CUDA(cudaEventCreateWithFlags(&ev_d2h[i], cudaEventDisableTiming));
    }
    init = true;
    return MP_OK;
  }
  int reserve(size_t bytes) {
    if (bytes <= buf_bytes)
      return MP_OK;
    if (buf) {
      cudaFree(buf);
      buf = nullptr;
      buf_bytes = 0;
    }
    MP_CUDA(cudaMalloc(&buf, bytes));
    buf_bytes = bytes;
    return MP_OK;
  }
  int reserve_pinned(size_t bytes) {
    if (bytes <= pin_bytes)
      return MP_OK;
    if (pin) {
      cudaFreeHost(pin);
      pin = nullptr;
      pin_bytes = 0;
    }
    MP_CUDA(cudaHostAlloc(&pin, bytes, cudaHostAllocDefault));
    pin_bytes = bytes;
    return MP_OK;
  }
};

HostPipe &host_pipe(int device) {
  static HostPipe pipes[64];
  return pipes[device & 63];
}

template <class KT>
uint64_t host_diag_search(const typename KT::T *a, uint64_t na,
                          const typename KT::T *b, uint64_t nb, uint64_t d) {
  uint64_t lo = d > nb ? d - nb : 0;
  uint64_t hi = d < na ? d : na;
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (KT::less(b[d - 1 - mid], a[mid]))  // core.hpp:110, ties to A
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

template <class KT, bool VALS>
int merge_host_pipelined(const void *a_, const uint32_t *av, uint64_t na,
                         const void *b_, const uint32_t *bv, uint64_t nb,
                         void *out_, uint32_t *outv, int device) {
  using T = typename KT::T;
  constexpr uint64_t ks = sizeof(T);
  const T *a = static_cast<const T *>(a_);
  const T *b = static_cast<const T *>(b_);
  T *out = static_cast<T *>(out_);
  const uint64_t n = na + nb;
  if (n == 0)
    return MP_OK;
  HostPipe &P = host_pipe(device);
  std::lock_guard<std::mutex> lk(P.mu);
  if (int rc = P.setup())
    return rc;
  // ~64 MiB of keys per chunk; never more chunks than needed
  // 64 MiB of keys per chunk by default (MP_HOST_CHUNK_MB overrides;
  // B200 A/B: 16 MiB 54.5 ms, 64 MiB 49.9 ms, 256 MiB 52.3 ms for config 2)
  static const uint64_t chunk_bytes = [] {
    const char *e = std::getenv("MP_HOST_CHUNK_MB");
    const long v = e ? std::atol(e) : 64;
    return static_cast<uint64_t>(v > 0 ? v : 64) << 20;
  }();
  const uint64_t Q = std::max<uint64_t>(1, std::min<uint64_t>(n, chunk_bytes / ks));
  // chunk boundaries: sizes ramp Q/8, Q/4, Q/2, then Q, and mirror at the
  // end, so the pipeline fill (first H2D) and drain (last D2H) are short
  std::vector<uint64_t> bounds{0};
  {
    std::vector<uint64_t> head, tail;
    uint64_t lo = 0, hi = n;
    for (uint64_t q = std::max<uint64_t>(1, Q / 8); q < Q && hi - lo > 2 * q; q *= 2) {
      head.push_back(q);
      tail.push_back(q);
      lo += q;
      hi -= q;
    }
    for (uint64_t q : head)
      bounds.push_back(bounds.back() + q);
    while (n - bounds.back() > (n - hi) + Q)
      bounds.push_back(bounds.back() + Q);
    bounds.push_back(hi);
    for (auto it = tail.rbegin(); it != tail.rend(); ++it)
      bounds.push_back(bounds.back() + *it);
    if (bounds.back() != n)
      bounds.push_back(n);
    std::vector<uint64_t> clean{0};
    for (size_t k = 1; k < bounds.size(); ++k)
      if (bounds[k] > clean.back())
        clean.push_back(bounds[k]);
    bounds.swap(clean);
  }
  const uint64_t chunks = bounds.size() - 1;
  auto up = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  // H2D copies start and end on 4 KiB host boundaries (the chunk's A and B
  // ranges widened by < 4 KiB each side): B200 A/B, config 2 with 64 MiB
  // chunks, copies alone: 50.2 ms at arbitrary element offsets vs 44.7 ms
  // for page-aligned DMA sources (tools/pipe_model.py).
  constexpr uint64_t kAlign = 4096;
  const uint64_t QA = Q + 2 * kAlign / ks;  // widened chunk capacity
  const uint64_t o_a = 0, o_b = up(QA * ks), o_o = o_b + up(QA * ks);
  const uint64_t o_av = o_o + up(Q * ks);
  const uint64_t o_bv = o_av + (VALS ? up(QA * 4) : 0);
  const uint64_t o_ov = o_bv + (VALS ? up(QA * 4) : 0);
  const uint64_t o_ws = o_ov + (VALS ? up(Q * 4) : 0);
  const uint64_t slot_bytes = o_ws + up(merge_ws_bytes<KT>(Q));
  if (int rc = P.reserve(slot_bytes * kSlots))
    return rc;
  // Pageable spans are staged through pinned host slots (CopyPool): chunk
  // k's inputs are copied into pinned slot k % kSlots before its H2D copies
  // are issued, and its output is copied out of the pinned slot after its
  // D2H copy landed -- one chunk later, so the copy engines and the merge
  // of chunk k overlap the host copies of chunks k - 1 and k + 1.
  const bool stage_in = is_pageable(a) || is_pageable(b) ||
                        (VALS && (is_pageable(av) || is_pageable(bv)));
  const bool stage_out = is_pageable(out) || (VALS && is_pageable(outv));
  // pinned slot layout: widened A, B (+ values) ranges, then the output
  const uint64_t pi_a = 0, pi_b = up(QA * ks) + kAlign;
  const uint64_t pi_av = pi_b + up(QA * ks) + kAlign;
  const uint64_t pi_bv = pi_av + (VALS ? up(QA * 4) + kAlign : 0);
  const uint64_t pi_o = pi_bv + (VALS ? up(QA * 4) + kAlign : 0);
  const uint64_t pi_ov = pi_o + up(Q * ks);
  const uint64_t pin_slot = (pi_ov + (VALS ? up(Q * 4) : 0) + kAlign - 1) & ~(kAlign - 1);
  if (stage_in || stage_out)
    if (int rc = P.reserve_pinned(pin_slot * kSlots))
      return rc;
  std::vector<std::tuple<void *, const void *, size_t>> jobs;
  auto drain = [&](uint64_t j) -> int {  // chunk j's output: pinned -> caller
    const int sj = static_cast<int>(j % kSlots);
    const char *pin = static_cast<const char *>(P.pin) + sj * pin_slot;
    MP_CUDA(cudaEventSynchronize(P.ev_d2h[sj]));
    const uint64_t e0 = bounds[j], e1 = bounds[j + 1];
    jobs.clear();
    jobs.emplace_back(out + e0, pin + pi_o, (e1 - e0) * ks);
    if (VALS)
      jobs.emplace_back(outv + e0, pin + pi_ov, (e1 - e0) * 4);
    CopyPool::get().copy(jobs);
    return MP_OK;
  };
  // [lo, lo + cnt) of a host array widened to 4 KiB boundaries (clamped to
  // the array, whole elements): {first byte, bytes, element shift of lo}
  struct Span {
    uintptr_t wb;
    uint64_t bytes;
    int64_t shift;
  };
  auto widen = [&](const void *src, uint64_t lo, uint64_t cnt, uint64_t total,
                   uint64_t es) -> Span {
    if (!cnt)
      return {0, 0, 0};
    const uintptr_t s0 = reinterpret_cast<uintptr_t>(src);
    const uintptr_t beg = s0 + lo * es, end = s0 + (lo + cnt) * es;
    uintptr_t wb = beg & ~uintptr_t(kAlign - 1);
    uintptr_t we = (end + kAlign - 1) & ~uintptr_t(kAlign - 1);
    wb = wb < s0 ? s0 + ((beg - s0) % es) : wb;
    wb = beg - ((beg - wb) / es) * es;  // whole elements before lo
    we = we > s0 + total * es ? s0 + total * es : we;
    we = end + ((we - end) / es) * es;
    return {wb, we - wb, static_cast<int64_t>((beg - wb) / es)};
  };
  uint64_t a_lo = 0;  // split of chunk k's start
  for (uint64_t k = 0; k < chunks; ++k) {
    const int s = static_cast<int>(k % kSlots);
    char *base = static_cast<char *>(P.buf) + s * slot_bytes;
    char *pin = (stage_in || stage_out) ? static_cast<char *>(P.pin) + s * pin_slot : nullptr;
    const uint64_t d0 = bounds[k], d1 = bounds[k + 1];
    const uint64_t a_hi = d1 == n ? na : host_diag_search<KT>(a, na, b, nb, d1);
    const uint64_t ca = a_hi - a_lo, cb = (d1 - a_hi) - (d0 - a_lo);
    const uint64_t b_lo = d0 - a_lo;
    if (k >= kSlots)  // the slot's previous chunk has left the device
      MP_CUDA(cudaStreamWaitEvent(P.h2d, P.ev_d2h[s], 0));
    const Span spans[4] = {widen(a, a_lo, ca, na, ks), widen(b, b_lo, cb, nb, ks),
                           VALS ? widen(av, a_lo, ca, na, 4) : Span{0, 0, 0},
                           VALS ? widen(bv, b_lo, cb, nb, 4) : Span{0, 0, 0}};
    const uint64_t dev_off[4] = {o_a, o_b, o_av, o_bv};
    const uint64_t pin_off[4] = {pi_a, pi_b, pi_av, pi_bv};
    const void *from[4];
    if (stage_in) {
      if (k >= kSlots)  // the slot's pinned inputs were last read by chunk k - kSlots
        MP_CUDA(cudaEventSynchronize(P.ev_h2d[s]));
      jobs.clear();
      for (int r = 0; r < 4; ++r) {
        // pinned copy at the same offset mod 4 KiB (page-aligned DMA source)
        char *p = pin + pin_off[r] + (spans[r].wb & (kAlign - 1));
        from[r] = p;
        if (spans[r].bytes)
          jobs.emplace_back(p, reinterpret_cast<const void *>(spans[r].wb), spans[r].bytes);
      }
      CopyPool::get().copy(jobs);
    } else {
      for (int r = 0; r < 4; ++r)
        from[r] = reinterpret_cast<const void *>(spans[r].wb);
    }
    for (int r = 0; r < (VALS ? 4 : 2); ++r)
      if (spans[r].bytes)
        MP_CUDA(cudaMemcpyAsync(base + dev_off[r], from[r], spans[r].bytes,
                                cudaMemcpyHostToDevice, P.h2d));
    const int64_t sa = spans[0].shift, sb = spans[1].shift;
    const int64_t sav = spans[2].shift, sbv = spans[3].shift;
    MP_CUDA(cudaEventRecord(P.ev_h2d[s], P.h2d));
    MP_CUDA(cudaStreamWaitEvent(P.cmp, P.ev_h2d[s], 0));
    uint64_t *ws = reinterpret_cast<uint64_t *>(base + o_ws);
    const T *da = reinterpret_cast<const T *>(base + o_a) + sa;
    const T *db = reinterpret_cast<const T *>(base + o_b) + sb;
    if (int rc = merge_plan<KT>(da, ca, db, cb, ws, P.cmp))
      return rc;
    if (int rc = merge_exec<KT, VALS, false>(
            da, VALS ? reinterpret_cast<uint32_t *>(base + o_av) + sav : nullptr,
            ca, db,
            VALS ? reinterpret_cast<uint32_t *>(base + o_bv) + sbv : nullptr, cb,
            base + o_o, VALS ? reinterpret_cast<uint32_t *>(base + o_ov) : nullptr,
            nullptr, ws, P.cmp))
      return rc;
    MP_CUDA(cudaEventRecord(P.ev_cmp[s], P.cmp));
    MP_CUDA(cudaStreamWaitEvent(P.d2h, P.ev_cmp[s], 0));
    void *to = stage_out ? static_cast<void *>(pin + pi_o) : static_cast<void *>(out + d0);
    MP_CUDA(cudaMemcpyAsync(to, base + o_o, (d1 - d0) * ks, cudaMemcpyDeviceToHost, P.d2h));
    if (VALS) {
      void *tov = stage_out ? static_cast<void *>(pin + pi_ov) : static_cast<void *>(outv + d0);
      MP_CUDA(cudaMemcpyAsync(tov, base + o_ov, (d1 - d0) * 4, cudaMemcpyDeviceToHost, P.d2h));
    }
    MP_CUDA(cudaEventRecord(P.ev_d2h[s], P.d2h));
    // drain two chunks behind: chunk k - 2's D2H has landed by now, so the
    // host never waits on the copy engines (kSlots >= 3 keeps k's slot free)
    if (stage_out && k >= kDrainLag)
      if (int rc = drain(k - kDrainLag))
        return rc;
    a_lo = a_hi;
  }
  if (stage_out)
    for (uint64_t j = chunks > kDrainLag ? chunks - kDrainLag : 0; j < chunks; ++j)
      if (int rc = drain(j))
        return rc;
  MP_CUDA(cudaStreamSynchronize(P.d2h));
  return MP_OK;
}

template <class KT> struct MergeHostOp {
  static int run(const void *a, const uint32_t *av, uint64_t na, const void *b,
                 const uint32_t *bv, uint64_t nb, void *out, uint32_t *outv,
                 int device) {
    if (av || bv || outv) {
      if (KT::kind == kElement)
        return fail(MP_ERR_UNSUPPORTED, "ELEMENT keys carry their own tag");
      return merge_host_pipelined<KT, true>(a, av, na, b, bv, nb, out, outv,
                                            device);
    }
    return merge_host_pipelined<KT, false>(a, nullptr, na, b, nullptr, nb, out,
                                           nullptr, device);
  }
};

}  // namespace

extern "C" {

const char *mp_last_error(void) { return g_err.c_str(); }
int mp_abi_version(void) { return 100; }
uint64_t mp_launch_count(void) { return g_launches.load(); }
uint64_t mp_key_size(int key_type) { return key_size(key_type); }

int mp_partition(int kt, const void *a, uint64_t na, const void *b,
                 uint64_t nb, uint64_t p, uint64_t *a_offs,
                 uint64_t *comparisons, void *stream) {
  g_err.clear();
  if (p == 0)
    return fail(MP_ERR_INVALID, "partition: p must be positive");
  if (!a_offs)
    return fail(MP_ERR_INVALID, "partition: a_offs is NULL");
  return dispatch<PartitionOp>(kt, a, na, b, nb, p, a_offs, comparisons,
                               static_cast<cudaStream_t>(stream));
}

int mp_diagonal_search(int kt, const void *a, uint64_t na, const void *b,
                       uint64_t nb, const uint64_t *diags, uint64_t count,
                       uint64_t *a_offs, uint64_t *comparisons, void *stream) {
  g_err.clear();
  if (count && (!diags || !a_offs))
    return fail(MP_ERR_INVALID, "diagonal_search: NULL array");
  return dispatch<DiagonalsOp>(kt, a, na, b, nb, diags, count, a_offs,
                               comparisons, static_cast<cudaStream_t>(stream));
}

int mp_merge(int kt, const void *a, const uint32_t *a_vals, uint64_t na,
             const void *b, const uint32_t *b_vals, uint64_t nb, void *out,
             uint32_t *out_vals, void *stream) {
  g_err.clear();
  if ((na && !a) || (nb && !b) || ((na + nb) && !out))
    return fail(MP_ERR_INVALID, "merge: NULL array");
  return dispatch<MergeOp>(kt, a, a_vals, na, b, b_vals, nb, out, out_vals, 0,
                           static_cast<uint64_t *>(nullptr),
                           static_cast<cudaStream_t>(stream));
}

uint64_t mp_merge_workspace_bytes(int kt, uint64_t na, uint64_t nb) {
  uint64_t out = 0;
  if (dispatch<MergeWsOp>(kt, na + nb, &out) != MP_OK)
    return 0;
  return out;
}

int mp_merge_plan(int kt, const void *a, uint64_t na, const void *b,
                  uint64_t nb, void *workspace, void *stream) {
  g_err.clear();
  if ((na && !a) || (nb && !b) || ((na + nb) && !workspace))
    return fail(MP_ERR_INVALID, "merge_plan: NULL array");
  return dispatch<MergeOp>(kt, a, static_cast<const uint32_t *>(nullptr), na,
                           b, static_cast<const uint32_t *>(nullptr), nb,
                           static_cast<void *>(nullptr),
                           static_cast<uint32_t *>(nullptr), 1,
                           static_cast<uint64_t *>(workspace),
                           static_cast<cudaStream_t>(stream));
}

int mp_merge_execute(int kt, const void *a, const uint32_t *a_vals,
                     uint64_t na, const void *b, const uint32_t *b_vals,
                     uint64_t nb, void *out, uint32_t *out_vals,
                     const void *workspace, void *stream) {
  g_err.clear();
  if ((na && !a) || (nb && !b) || ((na + nb) && (!out || !workspace)))
    return fail(MP_ERR_INVALID, "merge_execute: NULL array");
  return dispatch<MergeOp>(kt, a, a_vals, na, b, b_vals, nb, out, out_vals, 2,
                           const_cast<uint64_t *>(
                               static_cast<const uint64_t *>(workspace)),
                           static_cast<cudaStream_t>(stream));
}

int mp_merge_checksum(int kt, const void *a, uint64_t na, const void *b,
                      uint64_t nb, uint64_t *sum, void *stream) {
  g_err.clear();
  if ((na && !a) || (nb && !b) || !sum)
    return fail(MP_ERR_INVALID, "merge_checksum: NULL array");
  return dispatch<ChecksumOp>(kt, a, na, b, nb, sum,
                              static_cast<cudaStream_t>(stream));
}

uint64_t mp_sort_scratch_bytes(int kt, int with_vals, uint64_t n) {
  uint64_t out = 0;
  if (dispatch<ScratchOp>(kt, with_vals != 0, n, &out) != MP_OK)
    return 0;
  return out;
}

int mp_sort(int kt, void *keys, uint32_t *vals, uint64_t n, void *scratch,
            uint64_t scratch_bytes, void *stream) {
  g_err.clear();
  if (n && !keys)
    return fail(MP_ERR_INVALID, "sort: NULL keys");
  return dispatch<SortOp>(kt, static_cast<const void *>(keys),
                          static_cast<const uint32_t *>(vals), keys, vals, n,
                          scratch, scratch_bytes,
                          static_cast<cudaStream_t>(stream));
}

int mp_sort_to(int kt, const void *keys_in, const uint32_t *vals_in,
               void *keys_out, uint32_t *vals_out, uint64_t n, void *scratch,
               uint64_t scratch_bytes, void *stream) {
  g_err.clear();
  if (n && (!keys_in || !keys_out))
    return fail(MP_ERR_INVALID, "sort: NULL keys");
  return dispatch<SortOp>(kt, keys_in, vals_in, keys_out, vals_out, n, scratch,
                          scratch_bytes, static_cast<cudaStream_t>(stream));
}

int mp_merge_pieces(int kt, const mp_piece *a, int na_pieces,
                    const mp_piece *b, int nb_pieces, uint64_t out_begin,
                    uint64_t out_end, void *out, uint32_t *out_vals,
                    void *stream) {
  g_err.clear();
  if (!a || !b || ((out_end > out_begin) && !out))
    return fail(MP_ERR_INVALID, "merge_pieces: NULL array");
  return dispatch<PiecesOp>(kt, a, na_pieces, b, nb_pieces, out_begin, out_end,
                            out, out_vals, static_cast<cudaStream_t>(stream));
}

int mp_multi_merge(int kt, const mp_shard *a, int na, const mp_shard *b, int nb,
                   const mp_shard *out, int nout, void *const *streams) {
  g_err.clear();
  if (!a || !b || !out)
    return fail(MP_ERR_INVALID, "multi_merge: NULL shard table");
  return dispatch<MultiMergeOp>(kt, a, na, b, nb, out, nout, streams);
}

int mp_multi_sort(int kt, const mp_shard *shards, int P, void *const *streams) {
  g_err.clear();
  if (!shards)
    return fail(MP_ERR_INVALID, "multi_sort: NULL shard table");
  return dispatch<MultiSortOp>(kt, shards, P, streams);
}

int mp_pieces_partition(int kt, const mp_piece *a, int na_pieces, const mp_piece *b,
                        int nb_pieces, const uint64_t *diags, uint64_t count,
                        uint64_t *a_offs, void *stream) {
  g_err.clear();
  return dispatch<PiecesDiagOp>(kt, a, na_pieces, b, nb_pieces, diags, count, a_offs,
                                static_cast<cudaStream_t>(stream));
}

int mp_peer_copy(void *dst, const void *src, uint64_t bytes, void *stream) {
  g_err.clear();
  if (bytes == 0)
    return MP_OK;
  if (!dst || !src || (bytes & 15) || (reinterpret_cast<uintptr_t>(dst) & 15) ||
      (reinterpret_cast<uintptr_t>(src) & 15))
    return fail(MP_ERR_INVALID, "peer_copy: 16-byte aligned pointers and size required");
  int dev = 0, sms = 148;
  MP_CUDA(cudaGetDevice(&dev));
  MP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const uint64_t n16 = bytes / 16;
  const unsigned grid = static_cast<unsigned>(
      std::min<uint64_t>(uint64_t(sms) * 4, cdiv(n16, 4 * 512)));
  lsu_copy_kernel<<<grid ? grid : 1, 512, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint4 *>(dst), static_cast<const uint4 *>(src), n16);
  MP_LAUNCHED("lsu_copy_kernel");
  return MP_OK;
}

// ---- CUDA IPC (shards of other processes / GPUs) ---------------------------
int mp_ipc_export(const void *dev_ptr, void *handle64, uint64_t *offset) {
  g_err.clear();
  if (!dev_ptr || !handle64 || !offset)
    return fail(MP_ERR_INVALID, "ipc_export: NULL argument");
  // base of the allocation containing dev_ptr
  uintptr_t base = 0;
  size_t size = 0;
  if (!alloc_range(dev_ptr, &base, &size))
    return fail(MP_ERR_INVALID, "ipc_export: not a device allocation");
  cudaIpcMemHandle_t h;
  MP_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)));
  std::memcpy(handle64, &h, sizeof h);
  *offset = reinterpret_cast<unsigned long long>(dev_ptr) - base;
  return MP_OK;
}

// Imported mappings, one per (importing device, allocation handle), with a
// reference count: every mp_ipc_import takes a reference, mp_ipc_close drops
// one and unmaps the allocation when the last reference goes.
int mp_ipc_import(const void *handle64, uint64_t offset, void **dev_ptr) {
  g_err.clear();
  if (!handle64 || !dev_ptr)
    return fail(MP_ERR_INVALID, "ipc_import: NULL argument");
  int dev = 0;
  MP_CUDA(cudaGetDevice(&dev));
  const std::string key(static_cast<const char *>(handle64), sizeof(cudaIpcMemHandle_t));
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  for (auto &e : g_ipc)
    if (e.dev == dev && e.handle == key) {
      ++e.refs;
      *dev_ptr = static_cast<char *>(e.base) + offset;
      return MP_OK;
    }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof h);
  void *base = nullptr;
  MP_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  uintptr_t rb = 0;
  size_t rsz = 0;
  if (!alloc_range(base, &rb, &rsz) || rb != reinterpret_cast<uintptr_t>(base))
    rsz = 0;  // unknown extent: only the base pointer itself is recognised
  g_ipc.push_back({dev, key, base, rsz ? rsz : 1, 1});
  *dev_ptr = static_cast<char *>(base) + offset;
  return MP_OK;
}

int mp_ipc_close(const void *dev_ptr) {
  g_err.clear();
  if (!dev_ptr)
    return MP_OK;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  // the mapping whose base is the closest at or below dev_ptr
  size_t best = g_ipc.size();
  for (size_t k = 0; k < g_ipc.size(); ++k)
    if (g_ipc[k].base <= dev_ptr &&
        (best == g_ipc.size() || g_ipc[k].base > g_ipc[best].base))
      best = k;
  if (best == g_ipc.size())
    return fail(MP_ERR_INVALID, "ipc_close: not an imported mapping");
  if (--g_ipc[best].refs == 0) {
    DeviceScope ds(g_ipc[best].dev);
    const cudaError_t e = cudaIpcCloseMemHandle(g_ipc[best].base);
    g_ipc.erase(g_ipc.begin() + static_cast<long>(best));
    if (e != cudaSuccess)
      return cuda_fail(e, "cudaIpcCloseMemHandle");
  }
  return MP_OK;
}

// ---- stream-ordered flags (cross-process / cross-GPU ordering) ------------
// cuStreamWriteValue64 / cuStreamWaitValue64 through the runtime's driver
// entry points (no link-time libcuda dependency).  The write carries a
// system-scope fence (prior work of the stream is visible first); the wait
// blocks the stream's front end -- no SM is spent spinning.
namespace {
__global__ void signal_kernel(unsigned long long *flag, unsigned long long value) {
  // prior kernels of the stream are complete; order this store after them
  // for every observer, including peers over NVLink
  asm volatile("fence.sc.sys;\n\tst.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value)
               : "memory");
}
using StreamValueFn = int (*)(void *, unsigned long long, unsigned long long, unsigned int);
StreamValueFn driver_fn(const char *name) {
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return reinterpret_cast<StreamValueFn>(fn);
}
}  // namespace

int mp_signal(uint64_t *flag, uint64_t value, void *stream) {
  g_err.clear();
  static const StreamValueFn w = driver_fn("cuStreamWriteValue64");
  if (!flag || (reinterpret_cast<uintptr_t>(flag) & 7))
    return fail(MP_ERR_INVALID, "signal: flag must be an 8-byte aligned device address");
  // MP_SIGNAL_KERNEL=1: always the kernel path (tests it on any box)
  static const bool force_kernel = [] {
    const char *e = std::getenv("MP_SIGNAL_KERNEL");
    return e && std::strcmp(e, "1") == 0;
  }();
  if (!force_kernel && w && w(stream, reinterpret_cast<unsigned long long>(flag), value, 0) == 0)
    return MP_OK;
  // no stream memory operations on this address (e.g. a peer mapping the
  // driver refuses): one thread stores it, system-scope release
  cudaGetLastError();
  signal_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<unsigned long long *>(flag), value);
  MP_LAUNCHED("signal_kernel");
  return MP_OK;
}

int mp_wait(const uint64_t *flag, uint64_t value, void *stream) {
  g_err.clear();
  static const StreamValueFn w = driver_fn("cuStreamWaitValue64");
  if (!flag || (reinterpret_cast<uintptr_t>(flag) & 7))
    return fail(MP_ERR_INVALID, "wait: flag must be an 8-byte aligned device address");
  if (!w)
    return fail(MP_ERR_CUDA, "wait: cuStreamWaitValue64 unavailable");
  // CU_STREAM_WAIT_VALUE_GEQ (0): generation counters only grow
  if (int e = w(stream, reinterpret_cast<unsigned long long>(flag), value, 0))
    return fail(MP_ERR_CUDA, "cuStreamWaitValue64 failed (%d)", e);
  return MP_OK;
}

uint64_t mp_ipc_open_count(void) {
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  return g_ipc.size();
}

int mp_generate(int gen_kind, uint64_t seed, uint64_t first, uint64_t n,
                void *out, void *stream) {
  g_err.clear();
  if (gen_kind < 0 || gen_kind > 6)
    return fail(MP_ERR_INVALID, "generate: unknown kind %d", gen_kind);
  if (n == 0)
    return MP_OK;
  generate_kernel<<<static_cast<unsigned>(cdiv(n, 256)), 256, 0,
                    static_cast<cudaStream_t>(stream)>>>(gen_kind, seed, first,
                                                          n, out);
  MP_LAUNCHED("generate_kernel");
  return MP_OK;
}

// ---- host-buffer entry points ----------------------------------------------
}  // extern "C"

namespace {
// Stage host A and B (+ `extra` scratch bytes) into one device buffer.
struct HostInputs {
  ScratchGuard g;
  char *a = nullptr, *b = nullptr, *extra = nullptr;
  int stage(const void *ha, uint64_t na, const void *hb, uint64_t nb,
            uint64_t ks, uint64_t extra_bytes, cudaStream_t s) {
    const uint64_t ab = (na * ks + 255) & ~uint64_t(255);
    const uint64_t bb = (nb * ks + 255) & ~uint64_t(255);
    if (int rc = alloc_scratch(g, ab + bb + extra_bytes + 16, s))
      return rc;
    a = static_cast<char *>(g.p);
    b = a + ab;
    extra = b + bb;
    if (na)
      MP_CUDA(cudaMemcpyAsync(a, ha, na * ks, cudaMemcpyHostToDevice, s));
    if (nb)
      MP_CUDA(cudaMemcpyAsync(b, hb, nb * ks, cudaMemcpyHostToDevice, s));
    return MP_OK;
  }
};
}  // namespace

extern "C" {

int mp_partition_host(int kt, const void *a, uint64_t na, const void *b,
                      uint64_t nb, uint64_t p, uint64_t *a_offs,
                      uint64_t *comparisons, int device) {
  g_err.clear();
  const uint64_t ks = key_size(kt);
  if (!ks)
    return fail(MP_ERR_UNSUPPORTED, "unknown key type %d", kt);
  if (p == 0)
    return fail(MP_ERR_INVALID, "partition: p must be positive");
  if (!a_offs)
    return fail(MP_ERR_INVALID, "partition: a_offs is NULL");
  DeviceScope ds(device);
  if (ds.err != cudaSuccess)
    return cuda_fail(ds.err, "cudaSetDevice");
  cudaStream_t s = host_stream(device);
  HostInputs in;
  if (int rc = in.stage(a, na, b, nb, ks, (p + 2) * 8, s))
    return rc;
  uint64_t *offs = reinterpret_cast<uint64_t *>(in.extra);
  uint64_t *cnt = offs + p + 1;
  MP_CUDA(cudaMemsetAsync(cnt, 0, 8, s));
  if (int rc = mp_partition(kt, in.a, na, in.b, nb, p, offs, cnt, s))
    return rc;
  MP_CUDA(cudaMemcpyAsync(a_offs, offs, (p + 1) * 8, cudaMemcpyDeviceToHost, s));
  uint64_t c = 0;
  MP_CUDA(cudaMemcpyAsync(&c, cnt, 8, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  if (comparisons)
    *comparisons += c;
  return MP_OK;
}

int mp_diagonal_search_host(int kt, const void *a, uint64_t na, const void *b,
                            uint64_t nb, const uint64_t *diags, uint64_t count,
                            uint64_t *a_offs, uint64_t *comparisons,
                            int device) {
  g_err.clear();
  const uint64_t ks = key_size(kt);
  if (!ks)
    return fail(MP_ERR_UNSUPPORTED, "unknown key type %d", kt);
  if (count == 0)
    return MP_OK;
  if (!diags || !a_offs)
    return fail(MP_ERR_INVALID, "diagonal_search: NULL array");
  DeviceScope ds(device);
  if (ds.err != cudaSuccess)
    return cuda_fail(ds.err, "cudaSetDevice");
  cudaStream_t s = host_stream(device);
  HostInputs in;
  if (int rc = in.stage(a, na, b, nb, ks, (2 * count + 1) * 8, s))
    return rc;
  uint64_t *dd = reinterpret_cast<uint64_t *>(in.extra);
  uint64_t *offs = dd + count;
  uint64_t *cnt = offs + count;
  MP_CUDA(cudaMemcpyAsync(dd, diags, count * 8, cudaMemcpyHostToDevice, s));
  MP_CUDA(cudaMemsetAsync(cnt, 0, 8, s));
  if (int rc = mp_diagonal_search(kt, in.a, na, in.b, nb, dd, count, offs, cnt, s))
    return rc;
  MP_CUDA(cudaMemcpyAsync(a_offs, offs, count * 8, cudaMemcpyDeviceToHost, s));
  uint64_t c = 0;
  MP_CUDA(cudaMemcpyAsync(&c, cnt, 8, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  if (comparisons)
    *comparisons += c;
  return MP_OK;
}

uint64_t mp_segment_iterations(uint64_t na, uint64_t nb, uint64_t cache_elems) {
  if (cache_elems < 3)
    return 0;
  const uint64_t L = cache_elems / 3;
  return (na + nb + L - 1) / L;
}

int mp_segment_plan(int kt, const void *a, uint64_t na, const void *b,
                    uint64_t nb, uint64_t p, uint64_t cache_elems,
                    uint64_t *start_a, uint64_t *plan_comparisons,
                    uint64_t *merge_comparisons, void *stream) {
  g_err.clear();
  if (p == 0)
    return fail(MP_ERR_INVALID, "merge: worker count must be positive");
  if (cache_elems < 3)
    return fail(MP_ERR_INVALID, "merge: cache capacity must be at least 3");
  if ((na + nb) && !start_a)
    return fail(MP_ERR_INVALID, "segment_plan: NULL start array");
  return dispatch<SegmentOp>(kt, a, na, b, nb, p, cache_elems / 3, start_a,
                             plan_comparisons, merge_comparisons,
                             static_cast<uint64_t *>(nullptr),
                             static_cast<cudaStream_t>(stream));
}

int mp_segment_plan_host(int kt, const void *a, uint64_t na, const void *b,
                         uint64_t nb, uint64_t p, uint64_t cache_elems,
                         uint64_t *start_a, uint64_t *start_b,
                         uint64_t *plan_comparisons,
                         uint64_t *merge_comparisons, int device) {
  g_err.clear();
  const uint64_t ks = key_size(kt);
  if (!ks)
    return fail(MP_ERR_UNSUPPORTED, "unknown key type %d", kt);
  if (p == 0)
    return fail(MP_ERR_INVALID, "merge: worker count must be positive");
  if (cache_elems < 3)
    return fail(MP_ERR_INVALID, "merge: cache capacity must be at least 3");
  const uint64_t iters = mp_segment_iterations(na, nb, cache_elems);
  if (iters == 0)
    return MP_OK;
  if (!start_a)
    return fail(MP_ERR_INVALID, "segment_plan: NULL start array");
  DeviceScope ds(device);
  if (ds.err != cudaSuccess)
    return cuda_fail(ds.err, "cudaSetDevice");
  cudaStream_t s = host_stream(device);
  HostInputs in;
  if (int rc = in.stage(a, na, b, nb, ks, (iters + 2) * 8, s))
    return rc;
  uint64_t *st = reinterpret_cast<uint64_t *>(in.extra);
  uint64_t *cnt = st + iters;
  MP_CUDA(cudaMemsetAsync(cnt, 0, 16, s));
  if (int rc = mp_segment_plan(kt, in.a, na, in.b, nb, p, cache_elems, st, cnt,
                               cnt + 1, s))
    return rc;
  MP_CUDA(cudaMemcpyAsync(start_a, st, iters * 8, cudaMemcpyDeviceToHost, s));
  uint64_t c[2] = {0, 0};
  MP_CUDA(cudaMemcpyAsync(c, cnt, 16, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  const uint64_t L = cache_elems / 3;
  if (start_b)
    for (uint64_t k = 0; k < iters; ++k)
      start_b[k] = k * L - start_a[k];
  if (plan_comparisons)
    *plan_comparisons += c[0];
  if (merge_comparisons)
    *merge_comparisons += c[1];
  return MP_OK;
}

int mp_merge_host(int kt, const void *a, const uint32_t *av, uint64_t na,
                  const void *b, const uint32_t *bv, uint64_t nb, void *out,
                  uint32_t *outv, int device) {
  g_err.clear();
  const uint64_t ks = key_size(kt);
  if (!ks)
    return fail(MP_ERR_UNSUPPORTED, "unknown key type %d", kt);
  const uint64_t n = na + nb;
  if (n == 0)
    return MP_OK;
  if ((na && !a) || (nb && !b) || !out)
    return fail(MP_ERR_INVALID, "merge: NULL array");
  const bool vals = av || bv || outv;
  if (vals && (!outv || (na && !av) || (nb && !bv)))
    return fail(MP_ERR_INVALID, "values must be given for A, B and out");
  DeviceScope ds(device);
  if (ds.err != cudaSuccess)
    return cuda_fail(ds.err, "cudaSetDevice");
  return dispatch<MergeHostOp>(kt, a, av, na, b, bv, nb, out, outv, device);
}

int mp_merge_checksum_host(int kt, const void *a, uint64_t na, const void *b,
                           uint64_t nb, uint64_t *sum, int device) {
  g_err.clear();
  const uint64_t ks = key_size(kt);
  if (!ks)
    return fail(MP_ERR_UNSUPPORTED, "unknown key type %d", kt);
  if (!sum)
    return fail(MP_ERR_INVALID, "merge_checksum: NULL sum");
  DeviceScope ds(device);
  if (ds.err != cudaSuccess)
    return cuda_fail(ds.err, "cudaSetDevice");
  cudaStream_t s = host_stream(device);
  const uint64_t ab = (na * ks + 255) & ~uint64_t(255);
  const uint64_t bb = (nb * ks + 255) & ~uint64_t(255);
  ScratchGuard g;
  if (int rc = alloc_scratch(g, ab + bb + 256, s))
    return rc;
  char *d = static_cast<char *>(g.p);
  if (na)
    MP_CUDA(cudaMemcpyAsync(d, a, na * ks, cudaMemcpyHostToDevice, s));
  if (nb)
    MP_CUDA(cudaMemcpyAsync(d + ab, b, nb * ks, cudaMemcpyHostToDevice, s));
  uint64_t *dsum = reinterpret_cast<uint64_t *>(d + ab + bb);
  if (int rc = mp_merge_checksum(kt, d, na, d + ab, nb, dsum, s))
    return rc;
  MP_CUDA(cudaMemcpyAsync(sum, dsum, 8, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  return MP_OK;
}

}  // extern "C"

namespace {
// Host-buffer sort, pipelined over PCIe: the input is copied in chunks of
// C = 2^k block runs (~64 MiB) and each chunk is sorted on the device (the
// full mp_sort) while the next one is in flight -- a chunk-local sort leaves
// exactly the state the global bottom-up schedule has after log2(C/run)
// rounds (every aligned C-group sorted; stable within the group) -- then
// the remaining rounds run over the whole array and the result is copied
// out.  B200, 2^30 u32 keys: see DESIGN.md.
template <class KT, bool VALS>
int sort_host_pipelined(const void *keys_, const uint32_t *vals, uint64_t n,
                        void *out_keys, uint32_t *out_vals, int device,
                        bool *done) {
  using T = typename KT::T;
  constexpr uint64_t ks = sizeof(T);
  *done = false;
  const uint64_t run0 = sort_run0<KT, VALS>();
  if (run0 & (run0 - 1))
    return MP_OK;  // non-power-of-two runs (K3b): plain path
  uint64_t C = run0;
  while (C * 2 * ks <= (64ull << 20))
    C *= 2;
  if (n < 4 * C)
    return MP_OK;  // too small to pipeline: plain path
  HostPipe &hp = host_pipe(device);
  std::lock_guard<std::mutex> lk(hp.mu);
  if (int rc = hp.setup())
    return rc;
  const T *keys = static_cast<const T *>(keys_);
  auto up = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  const uint32_t NV = sort_round_tile<KT, VALS>();
  const SortLayout Lc = sort_layout<KT>(VALS, C);
  const uint64_t o_d = 0, o_aux = up(n * ks);
  const uint64_t o_dv = o_aux + up(n * ks);
  const uint64_t o_auxv = o_dv + (VALS ? up(n * 4) : 0);
  const uint64_t o_P = o_auxv + (VALS ? up(n * 4) : 0);
  const uint64_t o_cs = o_P + up((cdiv(n, NV) + 1) * 8);
  ScratchGuard g;
  if (int rc = alloc_scratch(g, o_cs + Lc.total, hp.cmp))
    return rc;
  char *base = static_cast<char *>(g.p);
  T *d = reinterpret_cast<T *>(base + o_d), *aux = reinterpret_cast<T *>(base + o_aux);
  uint32_t *dv = VALS ? reinterpret_cast<uint32_t *>(base + o_dv) : nullptr;
  uint32_t *auxv = VALS ? reinterpret_cast<uint32_t *>(base + o_auxv) : nullptr;
  uint64_t *P = reinterpret_cast<uint64_t *>(base + o_P);
  char *cs = base + o_cs;
  const uint64_t chunks = cdiv(n, C);
  // pageable spans: staged through the pinned slots (see the merge above)
  const bool stage_in = is_pageable(keys) || (VALS && is_pageable(vals));
  const bool stage_out = is_pageable(out_keys) || (VALS && is_pageable(out_vals));
  const uint64_t pin_v = up(C * ks), pin_slot = (pin_v + (VALS ? up(C * 4) : 0) + 4095) & ~4095ull;
  if (stage_in || stage_out)
    if (int rc = hp.reserve_pinned(pin_slot * kSlots))
      return rc;
  std::vector<std::tuple<void *, const void *, size_t>> jobs;
  for (uint64_t c = 0; c < chunks; ++c) {
    const int sl = static_cast<int>(c % kSlots);
    const uint64_t off = c * C, len = std::min<uint64_t>(C, n - off);
    const void *kin = keys + off, *vin = VALS ? vals + off : nullptr;
    if (stage_in) {
      char *pin = static_cast<char *>(hp.pin) + sl * pin_slot;
      if (c >= kSlots)  // the slot's previous H2D copy has read it
        MP_CUDA(cudaEventSynchronize(hp.ev_h2d[sl]));
      jobs.clear();
      jobs.emplace_back(pin, kin, len * ks);
      if (VALS)
        jobs.emplace_back(pin + pin_v, vin, len * 4);
      CopyPool::get().copy(jobs);
      kin = pin;
      vin = pin + pin_v;
    }
    MP_CUDA(cudaMemcpyAsync(d + off, kin, len * ks, cudaMemcpyHostToDevice, hp.h2d));
    if (VALS)
      MP_CUDA(cudaMemcpyAsync(dv + off, vin, len * 4, cudaMemcpyHostToDevice, hp.h2d));
    MP_CUDA(cudaEventRecord(hp.ev_h2d[sl], hp.h2d));
    MP_CUDA(cudaStreamWaitEvent(hp.cmp, hp.ev_h2d[sl], 0));
    if (int rc = sort_impl<KT, VALS>(d + off, VALS ? dv + off : nullptr, d + off,
                                     VALS ? dv + off : nullptr, len, cs, Lc.total, hp.cmp))
      return rc;
  }
  T *res = nullptr;
  uint32_t *resv = nullptr;
  if (int rc = sort_rounds_from<KT, VALS>(d, dv, aux, auxv, n, C, NV, P, hp.cmp, &res, &resv))
    return rc;
  if (!stage_out) {
    MP_CUDA(cudaMemcpyAsync(out_keys, res, n * ks, cudaMemcpyDeviceToHost, hp.cmp));
    if (VALS)
      MP_CUDA(cudaMemcpyAsync(out_vals, resv, n * 4, cudaMemcpyDeviceToHost, hp.cmp));
    MP_CUDA(cudaStreamSynchronize(hp.cmp));
    *done = true;
    return MP_OK;
  }
  // pageable output: chunk j lands in pinned slot j % kSlots (D2H stream)
  // and is copied out by the pool while chunk j + 1 is in flight
  MP_CUDA(cudaEventRecord(hp.ev_cmp[0], hp.cmp));
  MP_CUDA(cudaStreamWaitEvent(hp.d2h, hp.ev_cmp[0], 0));
  auto drain = [&](uint64_t j) -> int {
    const int sj = static_cast<int>(j % kSlots);
    const char *pin = static_cast<const char *>(hp.pin) + sj * pin_slot;
    const uint64_t off = j * C, len = std::min<uint64_t>(C, n - off);
    MP_CUDA(cudaEventSynchronize(hp.ev_d2h[sj]));
    jobs.clear();
    jobs.emplace_back(static_cast<T *>(out_keys) + off, pin, len * ks);
    if (VALS)
      jobs.emplace_back(out_vals + off, pin + pin_v, len * 4);
    CopyPool::get().copy(jobs);
    return MP_OK;
  };
  for (uint64_t j = 0; j < chunks; ++j) {
    const int sj = static_cast<int>(j % kSlots);
    char *pin = static_cast<char *>(hp.pin) + sj * pin_slot;
    const uint64_t off = j * C, len = std::min<uint64_t>(C, n - off);
    MP_CUDA(cudaMemcpyAsync(pin, res + off, len * ks, cudaMemcpyDeviceToHost, hp.d2h));
    if (VALS)
      MP_CUDA(cudaMemcpyAsync(pin + pin_v, resv + off, len * 4, cudaMemcpyDeviceToHost, hp.d2h));
    MP_CUDA(cudaEventRecord(hp.ev_d2h[sj], hp.d2h));
    if (j >= kDrainLag)
      if (int rc = drain(j - kDrainLag))
        return rc;
  }
  for (uint64_t j = chunks > kDrainLag ? chunks - kDrainLag : 0; j < chunks; ++j)
    if (int rc = drain(j))
      return rc;
  MP_CUDA(cudaStreamSynchronize(hp.d2h));
  *done = true;
  return MP_OK;
}

template <class KT> struct SortHostOp {
  static int run(const void *keys, const uint32_t *vals, uint64_t n,
                 void *out_keys, uint32_t *out_vals, int device, bool *done) {
    if (vals) {
      if (KT::kind == kElement)
        return fail(MP_ERR_UNSUPPORTED, "ELEMENT keys carry their own tag");
      return sort_host_pipelined<KT, true>(keys, vals, n, out_keys, out_vals, device, done);
    }
    return sort_host_pipelined<KT, false>(keys, nullptr, n, out_keys, nullptr, device, done);
  }
};
}  // namespace

extern "C" {

int mp_sort_host(int kt, const void *keys, const uint32_t *vals, uint64_t n,
                 void *out_keys, uint32_t *out_vals, int device) {
  g_err.clear();
  const uint64_t ks = key_size(kt);
  if (!ks)
    return fail(MP_ERR_UNSUPPORTED, "unknown key type %d", kt);
  if (n == 0)
    return MP_OK;
  if (!keys || !out_keys || (vals && !out_vals))
    return fail(MP_ERR_INVALID, "sort: NULL array");
  DeviceScope ds(device);
  if (ds.err != cudaSuccess)
    return cuda_fail(ds.err, "cudaSetDevice");
  static const bool pipe_env = [] {
    const char *e = std::getenv("MP_SORT_HOST_PIPE");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  if (pipe_env && (reinterpret_cast<uintptr_t>(keys) % ks) == 0 &&
      (reinterpret_cast<uintptr_t>(out_keys) % ks) == 0) {
    bool done = false;
    if (int rc = dispatch<SortHostOp>(kt, keys, vals, n, out_keys, out_vals, device, &done))
      return rc;
    if (done)
      return MP_OK;
  }
  cudaStream_t s = host_stream(device);
  const uint64_t kb = (n * ks + 255) & ~uint64_t(255);
  const uint64_t vb = vals ? ((n * 4 + 255) & ~uint64_t(255)) : 0;
  ScratchGuard g;
  if (int rc = alloc_scratch(g, kb + vb, s))
    return rc;
  char *d = static_cast<char *>(g.p);
  MP_CUDA(cudaMemcpyAsync(d, keys, n * ks, cudaMemcpyHostToDevice, s));
  uint32_t *dv = vals ? reinterpret_cast<uint32_t *>(d + kb) : nullptr;
  if (vals)
    MP_CUDA(cudaMemcpyAsync(dv, vals, n * 4, cudaMemcpyHostToDevice, s));
  if (int rc = mp_sort(kt, d, dv, n, nullptr, 0, s))
    return rc;
  MP_CUDA(cudaMemcpyAsync(out_keys, d, n * ks, cudaMemcpyDeviceToHost, s));
  if (vals)
    MP_CUDA(cudaMemcpyAsync(out_vals, dv, n * 4, cudaMemcpyDeviceToHost, s));
  MP_CUDA(cudaStreamSynchronize(s));
  return MP_OK;
}

void *mp_host_alloc(uint64_t bytes) {
  g_err.clear();
  void *p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
    cuda_fail(cudaGetLastError(), "cudaHostAlloc");
    return nullptr;
  }
  return p;
}

int mp_host_free(void *p) {
  g_err.clear();
  if (p)
    MP_CUDA(cudaFreeHost(p));
  return MP_OK;
}

int mp_release(int device) {
  g_err.clear();
  int count = 0;
  MP_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count || device >= 64)
    return fail(MP_ERR_INVALID, "release: no device %d", device);
  DeviceScope ds(device);
  if (ds.err != cudaSuccess)
    return cuda_fail(ds.err, "cudaSetDevice");
  MP_CUDA(cudaDeviceSynchronize());  // pending stream-ordered frees land
  HostPipe &P = host_pipe(device);
  {
    std::lock_guard<std::mutex> lk(P.mu);
    if (P.buf) {
      MP_CUDA(cudaFree(P.buf));
      P.buf = nullptr;
      P.buf_bytes = 0;
    }
    if (P.pin) {
      MP_CUDA(cudaFreeHost(P.pin));
      P.pin = nullptr;
      P.pin_bytes = 0;
    }
  }
  if (g_pools[device])
    MP_CUDA(cudaMemPoolTrimTo(g_pools[device], 0));
  return MP_OK;
}

}  // extern "C"

// key files (dataio.cpp:33-98) -> host / HBM
#include "mp_keyfile.cuh"
