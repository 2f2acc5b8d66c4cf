// C++ caller of the single-process multi-GPU entry points (no Python):
// mp_multi_merge and mp_multi_sort over a shard table, checked against
// std::merge / std::stable_sort on the host (the reference's own oracles,
// oracles.hpp:26-37).
//
//   test_multi_gpu [dev0 dev1 ...]     (default: 0 0 0 0 -- four shards on
//                                       GPU 0, the one-GPU lease)
//
// Exit code 0 = every case matched byte for byte.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <random>
#include <vector>

#include <cuda_runtime.h>

#include "mergepath_b200.h"

namespace {

int failures = 0;

#define CHECK(cond, ...)                                                       \
  do {                                                                         \
    if (!(cond)) {                                                             \
      std::fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__);                \
      std::fprintf(stderr, __VA_ARGS__);                                       \
      std::fprintf(stderr, "\n");                                              \
      ++failures;                                                              \
    }                                                                          \
  } while (0)

#define MP(x)                                                                  \
  do {                                                                         \
    const int rc_ = (x);                                                       \
    if (rc_ != MP_OK) {                                                        \
      std::fprintf(stderr, "%s -> %d: %s\n", #x, rc_, mp_last_error());        \
      std::exit(2);                                                            \
    }                                                                          \
  } while (0)

#define CU(x)                                                                  \
  do {                                                                         \
    const cudaError_t e_ = (x);                                                \
    if (e_ != cudaSuccess) {                                                   \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
      std::exit(2);                                                            \
    }                                                                          \
  } while (0)

struct DevBuf {  // one shard's device memory
  int dev = 0;
  void *p = nullptr;
  DevBuf(int d, size_t bytes) : dev(d) {
    CU(cudaSetDevice(d));
    CU(cudaMalloc(&p, bytes ? bytes : 16));
  }
  ~DevBuf() {
    cudaSetDevice(dev);
    cudaFree(p);
  }
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
};

std::vector<uint64_t> cuts(uint64_t n, int parts, std::mt19937_64 &rng, bool ragged) {
  std::vector<uint64_t> c(parts + 1, 0);
  for (int k = 1; k < parts; ++k)
    c[k] = ragged ? rng() % (n + 1) : k * n / parts;
  c[parts] = n;
  std::sort(c.begin(), c.end());
  return c;
}

// shards of x (keys + optional values) on the given devices
struct Sharded {
  std::vector<std::unique_ptr<DevBuf>> k, v;
  std::vector<mp_shard> tab;
};

template <class T>
Sharded upload(const std::vector<T> &x, const std::vector<uint32_t> *vals,
               const std::vector<uint64_t> &c, const std::vector<int> &devs) {
  Sharded s;
  for (size_t g = 0; g + 1 < c.size(); ++g) {
    const uint64_t len = c[g + 1] - c[g];
    const int d = devs[g % devs.size()];
    s.k.emplace_back(new DevBuf(d, len * sizeof(T)));
    CU(cudaMemcpy(s.k.back()->p, x.data() + c[g], len * sizeof(T), cudaMemcpyHostToDevice));
    uint32_t *vp = nullptr;
    if (vals) {
      s.v.emplace_back(new DevBuf(d, len * 4));
      CU(cudaMemcpy(s.v.back()->p, vals->data() + c[g], len * 4, cudaMemcpyHostToDevice));
      vp = static_cast<uint32_t *>(s.v.back()->p);
    }
    s.tab.push_back({d, s.k.back()->p, vp, len});
  }
  return s;
}

template <class T>
void download(const Sharded &s, std::vector<T> &x, std::vector<uint32_t> *vals) {
  uint64_t o = 0;
  for (const auto &sh : s.tab) {
    CU(cudaSetDevice(sh.device));
    CU(cudaMemcpy(x.data() + o, sh.keys, sh.len * sizeof(T), cudaMemcpyDeviceToHost));
    if (vals)
      CU(cudaMemcpy(vals->data() + o, sh.vals, sh.len * 4, cudaMemcpyDeviceToHost));
    o += sh.len;
  }
}

struct Kv {
  uint64_t k;
  uint32_t v;
};

void merge_case(const std::vector<int> &devs, uint64_t na, uint64_t nb, uint64_t keyspace,
                bool ragged, bool with_vals, bool async, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<uint64_t> a(na), b(nb);
  for (auto &x : a)
    x = rng() % keyspace;
  for (auto &x : b)
    x = rng() % keyspace;
  std::sort(a.begin(), a.end());
  std::sort(b.begin(), b.end());
  std::vector<uint32_t> av(na), bv(nb);
  std::iota(av.begin(), av.end(), 0u);
  for (uint64_t j = 0; j < nb; ++j)
    bv[j] = 0x80000000u | static_cast<uint32_t>(j);
  const int P = static_cast<int>(devs.size());
  Sharded A = upload(a, with_vals ? &av : nullptr, cuts(na, P, rng, ragged), devs);
  Sharded B = upload(b, with_vals ? &bv : nullptr, cuts(nb, P, rng, ragged), devs);
  std::vector<uint64_t> zero(na + nb, ~0ull);
  std::vector<uint32_t> zv(na + nb, 0);
  Sharded O = upload(zero, with_vals ? &zv : nullptr, cuts(na + nb, P, rng, ragged), devs);
  std::vector<cudaStream_t> st(P);
  if (async)
    for (int g = 0; g < P; ++g) {
      CU(cudaSetDevice(O.tab[g].device));
      CU(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    }
  MP(mp_multi_merge(MP_KEY_U64, A.tab.data(), P, B.tab.data(), P, O.tab.data(), P,
                    async ? reinterpret_cast<void *const *>(st.data()) : nullptr));
  if (async)
    for (int g = 0; g < P; ++g) {
      CU(cudaSetDevice(O.tab[g].device));
      CU(cudaStreamSynchronize(st[g]));
      CU(cudaStreamDestroy(st[g]));
    }
  std::vector<uint64_t> got(na + nb);
  std::vector<uint32_t> gotv(na + nb);
  download(O, got, with_vals ? &gotv : nullptr);
  // std::merge with a key-only comparator: stable, A first on ties
  std::vector<Kv> ka(na), kb(nb), want(na + nb);
  for (uint64_t i = 0; i < na; ++i)
    ka[i] = {a[i], av[i]};
  for (uint64_t j = 0; j < nb; ++j)
    kb[j] = {b[j], bv[j]};
  std::merge(ka.begin(), ka.end(), kb.begin(), kb.end(), want.begin(),
             [](const Kv &x, const Kv &y) { return x.k < y.k; });
  bool ok = true;
  for (uint64_t i = 0; i < na + nb && ok; ++i)
    ok = got[i] == want[i].k && (!with_vals || gotv[i] == want[i].v);
  CHECK(ok, "multi_merge na=%llu nb=%llu ragged=%d vals=%d async=%d", (unsigned long long)na,
        (unsigned long long)nb, ragged, with_vals, async);
}

void sort_case(const std::vector<int> &devs, uint64_t n, uint32_t keyspace, bool ragged,
               bool with_vals, bool async, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<uint32_t> x(n), v(n);
  for (auto &e : x)
    e = static_cast<uint32_t>(rng() % keyspace);
  std::iota(v.begin(), v.end(), 0u);
  const int P = static_cast<int>(devs.size());
  Sharded X = upload(x, with_vals ? &v : nullptr, cuts(n, P, rng, ragged), devs);
  std::vector<cudaStream_t> st(P);
  if (async)
    for (int g = 0; g < P; ++g) {
      CU(cudaSetDevice(X.tab[g].device));
      CU(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    }
  MP(mp_multi_sort(MP_KEY_U32, X.tab.data(), P,
                   async ? reinterpret_cast<void *const *>(st.data()) : nullptr));
  if (async)
    for (int g = 0; g < P; ++g) {
      CU(cudaSetDevice(X.tab[g].device));
      CU(cudaStreamSynchronize(st[g]));
      CU(cudaStreamDestroy(st[g]));
    }
  std::vector<uint32_t> got(n), gotv(n);
  download(X, got, with_vals ? &gotv : nullptr);
  std::vector<uint32_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0u);
  std::stable_sort(idx.begin(), idx.end(), [&](uint32_t i, uint32_t j) { return x[i] < x[j]; });
  bool ok = true;
  for (uint64_t i = 0; i < n && ok; ++i)
    ok = got[i] == x[idx[i]] && (!with_vals || gotv[i] == idx[i]);
  CHECK(ok, "multi_sort n=%llu P=%d ragged=%d vals=%d async=%d", (unsigned long long)n, P,
        ragged, with_vals, async);
}

}  // namespace

int main(int argc, char **argv) {
  std::vector<int> devs;
  for (int i = 1; i < argc; ++i)
    devs.push_back(std::atoi(argv[i]));
  if (devs.empty())
    devs = {0, 0, 0, 0};
  uint64_t seed = 1406;
  for (bool async : {false, true})
    for (bool vals : {false, true}) {
      merge_case(devs, 1000003, 777777, 1ull << 40, false, vals, async, seed++);
      merge_case(devs, 300000, 2000001, 64, true, vals, async, seed++);  // heavy ties
      merge_case(devs, 5, 131072, 1000, true, vals, async, seed++);
      sort_case(devs, 3000017, 1u << 31, false, vals, async, seed++);
      sort_case(devs, 1000001, 100, true, vals, async, seed++);  // stability visible
    }
  for (int P = 1; P <= static_cast<int>(devs.size()) + 3 && P <= 16; P += 2) {
    std::vector<int> d(P);
    for (int g = 0; g < P; ++g)
      d[g] = devs[g % devs.size()];
    sort_case(d, 200000 + P, 1000, true, true, P & 1, seed++);
    merge_case(d, 100000, 50000 + P, 5000, true, true, P & 1, seed++);
  }
  // argument errors
  mp_shard bad{0, nullptr, nullptr, 10};
  CHECK(mp_multi_sort(MP_KEY_U32, &bad, 1, nullptr) == MP_ERR_INVALID, "NULL keys accepted");
  CHECK(mp_multi_sort(MP_KEY_U32, &bad, 0, nullptr) == MP_ERR_INVALID, "P = 0 accepted");
  std::printf("%s: %d failure(s)\n", failures ? "FAIL" : "OK", failures);
  return failures ? 1 : 0;
}
