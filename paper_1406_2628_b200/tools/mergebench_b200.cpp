// mergebench_b200 -- the reference benchmark tool's command-line contract
// (SPEC.md module bench-cli; mergebench.cpp) on the B200 backend.
//
//   mergebench_b200 gen    --dist D --na N --nb N [--seed S] --out-a F --out-b F [--format bin|text]
//   mergebench_b200 merge  --a F --b F [--variant regular|segmented] [--threads 1,2,..]
//                          [--cache-elems C,..] [--reps R] [--sink memory|register]
//                          [--format json|csv] [--out F] [--residency device|host|file [--merged-out F]]
//                          [--host-memory pinned|pageable] [--device N]
//   mergebench_b200 sort   --in F [--variant plain|cache_efficient] [--threads ..]
//                          [--cache-elems C] [--reps R] [--format json|csv] [--out F]
//                          [--residency device|host|file [--sorted-out F]] [--host-memory pinned|pageable] [--device N]
//   mergebench_b200 report --in F [--format json|csv] [--out F]
//
// Same subcommands, flags, report rows {op, variant, n, p, cache_elems, reps,
// median_seconds, mean_seconds, speedup_vs_p1, partition_comparisons,
// merge_steps, merge_rounds, verified} and exit codes (0 ok, 1 usage, 2 I/O,
// 3 validation, 4 reference mismatch) as the reference.  Every timed
// repetition is checked against std::merge / std::sort of the same keys
// before its row is reported.  Key files are the reference's MPKB0001 /
// text formats (mp_keyfile_*).
//
// B200 specifics: keys are i64 (MP_KEY_I64).  --residency device (default)
// streams the key files into HBM once (mp_keyfile_load) and times the device
// call with CUDA events (mp_merge / mp_merge_checksum / mp_sort_to);
// --residency host times the drop-in template call on host spans with a
// steady clock, as the reference does (PCIe copies included); merge
// --residency file times mp_keyfile_merge (key files in, merged key file
// out, the ingest overlapped with the merge) and verifies the file; sort
// --residency file likewise with mp_keyfile_sort.  p only
// feeds the statistics, which are the reference's (device replays); the
// GPU grid does not depend on it.  `cachesim` models a CPU cache and is not
// part of this backend.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <numeric>
#include <optional>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include <cuda_runtime.h>

#include "mergepath/core.hpp"
#include "mergepath/parallel.hpp"
#include "mergepath/sort.hpp"
#include "mergepath_b200.h"

namespace {

// ---------------------------------------------------------------- errors --
struct usage_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct io_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct mismatch_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void check_status(int rc) {
  if (rc == MP_OK)
    return;
  const std::string msg = mp_last_error();
  if (rc == MP_ERR_INVALID)
    throw std::invalid_argument(msg);
  if (rc == MP_ERR_IO)
    throw io_error(msg);
  throw std::runtime_error("mergepath status " + std::to_string(rc) + ": " + msg);
}

void check_cuda(cudaError_t e, const char *what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ json --
// Just enough JSON for the report: null, bool, integers, doubles, strings,
// arrays and objects (insertion-ordered), with a writer and a parser.
struct Json {
  enum Kind { Null, Bool, Int, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  long long i = 0;
  double d = 0;
  std::string s;
  std::vector<Json> a;
  std::vector<std::pair<std::string, Json>> o;

  static Json null() { return Json(); }
  static Json boolean(bool v) { Json j; j.kind = Bool; j.b = v; return j; }
  static Json integer(long long v) { Json j; j.kind = Int; j.i = v; return j; }
  static Json number(double v) { Json j; j.kind = Num; j.d = v; return j; }
  static Json string(std::string v) { Json j; j.kind = Str; j.s = std::move(v); return j; }
  static Json array() { Json j; j.kind = Arr; return j; }
  static Json object() { Json j; j.kind = Obj; return j; }

  Json &set(const std::string &k, Json v) {
    for (auto &kv : o)
      if (kv.first == k) {
        kv.second = std::move(v);
        return *this;
      }
    o.emplace_back(k, std::move(v));
    return *this;
  }
  const Json *get(const std::string &k) const {
    for (const auto &kv : o)
      if (kv.first == k)
        return &kv.second;
    return nullptr;
  }
};

void dump_string(const std::string &s, std::ostream &out) {
  out << '"';
  for (unsigned char c : s) {
    switch (c) {
    case '"': out << "\\\""; break;
    case '\\': out << "\\\\"; break;
    case '\n': out << "\\n"; break;
    case '\t': out << "\\t"; break;
    case '\r': out << "\\r"; break;
    default:
      if (c < 0x20) {
        char buf[8];
        std::snprintf(buf, sizeof buf, "\\u%04x", c);
        out << buf;
      } else {
        out << c;
      }
    }
  }
  out << '"';
}

std::string fmt_double(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  std::string s = buf;
  if (s.find_first_of(".eEn") == std::string::npos)
    s += ".0";
  return s;
}

void dump(const Json &j, std::ostream &out, int indent, int depth) {
  const std::string pad(static_cast<size_t>(indent * (depth + 1)), ' ');
  const std::string pad0(static_cast<size_t>(indent * depth), ' ');
  switch (j.kind) {
  case Json::Null: out << "null"; break;
  case Json::Bool: out << (j.b ? "true" : "false"); break;
  case Json::Int: out << j.i; break;
  case Json::Num: out << fmt_double(j.d); break;
  case Json::Str: dump_string(j.s, out); break;
  case Json::Arr:
    if (j.a.empty()) { out << "[]"; break; }
    out << "[\n";
    for (size_t k = 0; k < j.a.size(); ++k) {
      out << pad;
      dump(j.a[k], out, indent, depth + 1);
      out << (k + 1 < j.a.size() ? ",\n" : "\n");
    }
    out << pad0 << ']';
    break;
  case Json::Obj:
    if (j.o.empty()) { out << "{}"; break; }
    out << "{\n";
    for (size_t k = 0; k < j.o.size(); ++k) {
      out << pad;
      dump_string(j.o[k].first, out);
      out << ": ";
      dump(j.o[k].second, out, indent, depth + 1);
      out << (k + 1 < j.o.size() ? ",\n" : "\n");
    }
    out << pad0 << '}';
    break;
  }
}

struct JsonParser {
  const std::string &t;
  size_t p = 0;
  explicit JsonParser(const std::string &text) : t(text) {}
  [[noreturn]] void bad(const char *why) {
    throw std::invalid_argument("bad report file: " + std::string(why) +
                                " at offset " + std::to_string(p));
  }
  void ws() {
    while (p < t.size() && std::isspace(static_cast<unsigned char>(t[p])))
      ++p;
  }
  bool lit(const char *w) {
    const size_t n = std::strlen(w);
    if (t.compare(p, n, w) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  std::string str() {
    if (t[p] != '"')
      bad("expected string");
    ++p;
    std::string s;
    while (p < t.size() && t[p] != '"') {
      char c = t[p++];
      if (c == '\\') {
        if (p >= t.size())
          bad("bad escape");
        const char e = t[p++];
        switch (e) {
        case 'n': s += '\n'; break;
        case 't': s += '\t'; break;
        case 'r': s += '\r'; break;
        case 'b': s += '\b'; break;
        case 'f': s += '\f'; break;
        case 'u': {
          if (p + 4 > t.size())
            bad("bad \\u escape");
          const unsigned v = static_cast<unsigned>(std::stoul(t.substr(p, 4), nullptr, 16));
          p += 4;
          if (v < 0x80) {
            s += static_cast<char>(v);
          } else if (v < 0x800) {
            s += static_cast<char>(0xC0 | (v >> 6));
            s += static_cast<char>(0x80 | (v & 0x3F));
          } else {
            s += static_cast<char>(0xE0 | (v >> 12));
            s += static_cast<char>(0x80 | ((v >> 6) & 0x3F));
            s += static_cast<char>(0x80 | (v & 0x3F));
          }
          break;
        }
        default: s += e;
        }
      } else {
        s += c;
      }
    }
    if (p >= t.size())
      bad("unterminated string");
    ++p;
    return s;
  }
  Json value() {
    ws();
    if (p >= t.size())
      bad("unexpected end");
    const char c = t[p];
    if (c == '{') {
      ++p;
      Json j = Json::object();
      ws();
      if (p < t.size() && t[p] == '}') { ++p; return j; }
      for (;;) {
        ws();
        std::string k = str();
        ws();
        if (p >= t.size() || t[p] != ':')
          bad("expected ':'");
        ++p;
        j.set(k, value());
        ws();
        if (p < t.size() && t[p] == ',') { ++p; continue; }
        if (p < t.size() && t[p] == '}') { ++p; return j; }
        bad("expected ',' or '}'");
      }
    }
    if (c == '[') {
      ++p;
      Json j = Json::array();
      ws();
      if (p < t.size() && t[p] == ']') { ++p; return j; }
      for (;;) {
        j.a.push_back(value());
        ws();
        if (p < t.size() && t[p] == ',') { ++p; continue; }
        if (p < t.size() && t[p] == ']') { ++p; return j; }
        bad("expected ',' or ']'");
      }
    }
    if (c == '"')
      return Json::string(str());
    if (lit("null")) return Json::null();
    if (lit("true")) return Json::boolean(true);
    if (lit("false")) return Json::boolean(false);
    const size_t b = p;
    if (p < t.size() && (t[p] == '-' || t[p] == '+'))
      ++p;
    bool real = false;
    while (p < t.size() && (std::isdigit(static_cast<unsigned char>(t[p])) ||
                            t[p] == '.' || t[p] == 'e' || t[p] == 'E' ||
                            t[p] == '-' || t[p] == '+')) {
      real |= t[p] == '.' || t[p] == 'e' || t[p] == 'E';
      ++p;
    }
    if (p == b)
      bad("unexpected character");
    const std::string num = t.substr(b, p - b);
    try {
      return real ? Json::number(std::stod(num)) : Json::integer(std::stoll(num));
    } catch (...) {
      bad("bad number");
    }
  }
};

Json parse_json(const std::string &text) {
  JsonParser ps(text);
  Json j = ps.value();
  ps.ws();
  if (ps.p != text.size())
    ps.bad("trailing content");
  return j;
}

// --------------------------------------------------------------- report --
struct Row {
  std::string op, variant;
  std::size_t n = 0, p = 0, cache_elems = 0, reps = 0;
  double median_seconds = 0, mean_seconds = 0;
  std::optional<double> speedup_vs_p1;
  std::optional<std::uint64_t> partition_comparisons, merge_steps;
  std::optional<std::size_t> merge_rounds;
  bool verified = false;
};

Json row_json(const Row &r) {
  auto opt_u = [](const auto &v) {
    return v ? Json::integer(static_cast<long long>(*v)) : Json::null();
  };
  Json j = Json::object();
  j.set("op", Json::string(r.op));
  j.set("variant", Json::string(r.variant));
  j.set("n", Json::integer(static_cast<long long>(r.n)));
  j.set("p", Json::integer(static_cast<long long>(r.p)));
  j.set("cache_elems", Json::integer(static_cast<long long>(r.cache_elems)));
  j.set("reps", Json::integer(static_cast<long long>(r.reps)));
  j.set("median_seconds", Json::number(r.median_seconds));
  j.set("mean_seconds", Json::number(r.mean_seconds));
  j.set("verified", Json::boolean(r.verified));
  j.set("speedup_vs_p1", r.speedup_vs_p1 ? Json::number(*r.speedup_vs_p1) : Json::null());
  j.set("partition_comparisons", opt_u(r.partition_comparisons));
  j.set("merge_steps", opt_u(r.merge_steps));
  j.set("merge_rounds", opt_u(r.merge_rounds));
  return j;
}

const char *kCsvCols[] = {"op", "variant", "n", "p", "cache_elems", "reps",
                          "median_seconds", "mean_seconds", "speedup_vs_p1",
                          "partition_comparisons", "merge_steps",
                          "merge_rounds", "verified"};

void render_csv(const Json &report, std::ostream &out) {
  for (size_t c = 0; c < std::size(kCsvCols); ++c)
    out << (c ? "," : "") << kCsvCols[c];
  out << '\n';
  const Json *rows = report.get("rows");
  for (const Json &r : rows->a) {
    for (size_t c = 0; c < std::size(kCsvCols); ++c) {
      if (c)
        out << ',';
      const Json *v = r.get(kCsvCols[c]);
      if (!v || v->kind == Json::Null)
        continue;
      switch (v->kind) {
      case Json::Num: {
        char buf[32];
        std::snprintf(buf, sizeof buf, "%.9g", v->d);
        out << buf;
        break;
      }
      case Json::Bool: out << (v->b ? "true" : "false"); break;
      case Json::Str: out << v->s; break;
      case Json::Int: out << v->i; break;
      default: dump(*v, out, 0, 0);
      }
    }
    out << '\n';
  }
}

void emit(const Json &report, const std::string &format, const std::string &path) {
  std::ofstream file;
  std::ostream *out = &std::cout;
  if (!path.empty()) {
    file.open(path);
    if (!file)
      throw io_error("cannot open for writing: " + path);
    out = &file;
  }
  if (format == "csv") {
    render_csv(report, *out);
  } else {
    dump(report, *out, 2, 0);
    *out << '\n';
  }
  out->flush();
  if (!*out)
    throw io_error("write failed");
}

// Row statistics of one configuration's timed repetitions: the row schema's
// median_seconds and mean_seconds (the reference tool's columns; the
// computation here is its own).
struct TimeStats {
  double median = 0, mean = 0;
};
TimeStats time_stats(std::vector<double> t) {
  TimeStats st;
  if (t.empty())
    return st;
  st.mean = std::accumulate(t.begin(), t.end(), 0.0) / static_cast<double>(t.size());
  const auto mid = t.begin() + static_cast<std::ptrdiff_t>(t.size() / 2);
  std::nth_element(t.begin(), mid, t.end());
  st.median = *mid;
  if (t.size() % 2 == 0)  // even count: average with the largest of the lower half
    st.median = 0.5 * (st.median + *std::max_element(t.begin(), mid));
  return st;
}

// speedup_vs_p1: each row's median against the p = 1 row of the same
// (op, variant, cache_elems) configuration, when that row exists.
void fill_speedups(std::vector<Row> &rows) {
  std::map<std::tuple<std::string, std::string, std::size_t>, double> p1;
  for (const Row &r : rows)
    if (r.p == 1)
      p1.emplace(std::make_tuple(r.op, r.variant, r.cache_elems), r.median_seconds);
  for (Row &r : rows) {
    const auto it = p1.find(std::make_tuple(r.op, r.variant, r.cache_elems));
    if (!r.speedup_vs_p1 && it != p1.end() && r.median_seconds > 0)
      r.speedup_vs_p1 = it->second / r.median_seconds;
  }
}

// Default worker sweep: powers of two up to the host's hardware threads,
// plus that count itself.
std::size_t host_threads() { return std::max(1u, std::thread::hardware_concurrency()); }
std::vector<std::size_t> thread_sweep() {
  const std::size_t hw = host_threads();
  std::vector<std::size_t> sweep;
  for (std::size_t p = 1; p < hw; p <<= 1)
    sweep.push_back(p);
  sweep.push_back(hw);
  return sweep;
}

// ---------------------------------------------------------------- args ----
struct Args {
  std::map<std::string, std::string> kv;
  std::vector<std::string> flags;
};

Args parse_args(int argc, char **argv, int first,
                const std::vector<std::string> &allowed) {
  Args a;
  for (int k = first; k < argc; ++k) {
    std::string s = argv[k];
    if (s.rfind("--", 0) != 0)
      throw usage_error("unexpected argument: " + s);
    std::string key = s.substr(2), val;
    const auto eq = key.find('=');
    if (eq != std::string::npos) {
      val = key.substr(eq + 1);
      key = key.substr(0, eq);
    } else {
      if (k + 1 >= argc)
        throw usage_error("--" + key + " needs a value");
      val = argv[++k];
    }
    if (std::find(allowed.begin(), allowed.end(), key) == allowed.end())
      throw usage_error("unknown option --" + key);
    a.kv[key] = val;
  }
  return a;
}

std::string need(const Args &a, const std::string &k) {
  auto it = a.kv.find(k);
  if (it == a.kv.end())
    throw usage_error("--" + k + " is required");
  return it->second;
}
std::string opt(const Args &a, const std::string &k, const std::string &def) {
  auto it = a.kv.find(k);
  return it == a.kv.end() ? def : it->second;
}
void member(const std::string &k, const std::string &v,
            std::initializer_list<const char *> ok) {
  for (const char *o : ok)
    if (v == o)
      return;
  throw usage_error("--" + k + ": '" + v + "' not allowed");
}
std::uint64_t to_u64(const std::string &k, const std::string &v) {
  if (v.empty() || v.find_first_not_of("0123456789") != std::string::npos)
    throw usage_error("--" + k + ": not a non-negative integer: " + v);
  try {
    return std::stoull(v);
  } catch (...) {
    throw usage_error("--" + k + ": out of range: " + v);
  }
}
std::vector<std::size_t> to_list(const std::string &k, const std::string &v) {
  std::vector<std::size_t> out;
  std::stringstream ss(v);
  std::string item;
  while (std::getline(ss, item, ','))
    out.push_back(static_cast<std::size_t>(to_u64(k, item)));
  return out;
}
std::size_t reps_of(const Args &a, std::size_t def) {
  const std::uint64_t r = to_u64("reps", opt(a, "reps", std::to_string(def)));
  if (r < 3 || r > 1000000)
    throw usage_error("--reps must be in [3, 1000000]");
  return static_cast<std::size_t>(r);
}

// ------------------------------------------------------------- key files --
std::vector<std::int64_t> read_keys(const std::string &path) {
  std::uint64_t n = 0;
  int bin = 0;
  check_status(mp_keyfile_count(path.c_str(), &n, &bin));
  std::vector<std::int64_t> v(n);
  std::uint64_t got = 0;
  check_status(mp_keyfile_read(path.c_str(), v.data(), n, &got));
  v.resize(got);
  return v;
}
std::vector<std::int64_t> load_sorted(const std::string &path, const char *role) {
  auto v = read_keys(path);
  if (!std::is_sorted(v.begin(), v.end()))
    throw std::invalid_argument(std::string(role) + " input is not sorted: " + path);
  return v;
}

// device buffer (RAII)
struct DevBuf {
  void *p = nullptr;
  explicit DevBuf(std::size_t bytes) {
    check_cuda(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc");
  }
  ~DevBuf() {
    if (p)
      cudaFree(p);
  }
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
};

struct Stream {
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  Stream() {
    check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    check_cuda(cudaEventCreate(&e0), "event");
    check_cuda(cudaEventCreate(&e1), "event");
  }
  ~Stream() {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
  }
  template <class F> double time(F &&f) {
    check_cuda(cudaEventRecord(e0, s), "event record");
    f();
    check_cuda(cudaEventRecord(e1, s), "event record");
    check_cuda(cudaEventSynchronize(e1), "event sync");
    float ms = 0;
    check_cuda(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
    return ms / 1e3;
  }
};

// Page-locks a host vector for the duration of a scope (host residency:
// the timed calls then stream through the PCIe pipeline without driver
// staging; registration happens before timing, like the reference's setup).
struct PinScope {
  void *p = nullptr;
  PinScope(void *ptr, std::size_t bytes) {
    if (ptr && bytes && cudaHostRegister(ptr, bytes, cudaHostRegisterDefault) == cudaSuccess)
      p = ptr;
    else
      cudaGetLastError();  // pageable fallback: still correct, slower
  }
  ~PinScope() {
    if (p)
      cudaHostUnregister(p);
  }
  PinScope(const PinScope &) = delete;
  PinScope &operator=(const PinScope &) = delete;
};

template <class F> double wall(F &&f) {
  const auto t0 = std::chrono::steady_clock::now();
  f();
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

std::string device_name(int dev) {
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess)
    return "?";
  return prop.name;
}

// ------------------------------------------------------------------ gen ---
// The reference's input generator (dataio.cpp:126-169), restated: uniform
// draws from a small key range (duplicates common), all keys equal,
// disjoint ranges (every A key above every B key), and interleaved evens /
// odds.  libstdc++'s mt19937_64 and uniform_int_distribution make the files
// byte-identical to the reference's for the same seed.
int run_gen(const Args &a) {
  const std::string dist = opt(a, "dist", "uniform");
  member("dist", dist, {"uniform", "all_equal", "disjoint_ranges", "interleaved"});
  const std::size_t na = static_cast<std::size_t>(to_u64("na", need(a, "na")));
  const std::size_t nb = static_cast<std::size_t>(to_u64("nb", need(a, "nb")));
  const std::uint64_t seed = to_u64("seed", opt(a, "seed", "1"));
  const std::string fa = need(a, "out-a"), fb = need(a, "out-b");
  const std::string format = opt(a, "format", "bin");
  member("format", format, {"bin", "text"});
  std::vector<std::int64_t> A(na), B(nb);
  if (dist == "uniform") {
    std::mt19937_64 rng(seed);
    const std::int64_t hi = static_cast<std::int64_t>(std::max<std::size_t>(4, (na + nb) / 2));
    std::uniform_int_distribution<std::int64_t> pick(0, hi - 1);
    for (auto &v : A)
      v = pick(rng);
    for (auto &v : B)
      v = pick(rng);
    std::sort(A.begin(), A.end());
    std::sort(B.begin(), B.end());
  } else if (dist == "all_equal") {
    std::fill(A.begin(), A.end(), 7);
    std::fill(B.begin(), B.end(), 7);
  } else if (dist == "disjoint_ranges") {
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<std::int64_t> low(0, (1 << 20) - 1);
    for (auto &v : B)
      v = low(rng);
    for (auto &v : A)
      v = (std::int64_t{1} << 40) + low(rng);
    std::sort(A.begin(), A.end());
    std::sort(B.begin(), B.end());
  } else {
    for (std::size_t i = 0; i < na; ++i)
      A[i] = static_cast<std::int64_t>(2 * i);
    for (std::size_t j = 0; j < nb; ++j)
      B[j] = static_cast<std::int64_t>(2 * j + 1);
  }
  const int bin = format == "bin";
  check_status(mp_keyfile_write(fa.c_str(), A.data(), A.size(), bin));
  check_status(mp_keyfile_write(fb.c_str(), B.data(), B.size(), bin));
  return 0;
}

int device_of(const Args &a) {
  const int dev = static_cast<int>(to_u64("device", opt(a, "device", "0")));
  check_cuda(cudaSetDevice(dev), "cudaSetDevice");
  mergepath::b200::set_device(dev);
  return dev;
}

// ---------------------------------------------------------------- merge ---
int run_merge(const Args &a) {
  const std::string fa = need(a, "a"), fb = need(a, "b");
  const std::string variant = opt(a, "variant", "regular");
  member("variant", variant, {"regular", "segmented"});
  const std::string sink = opt(a, "sink", "memory");
  member("sink", sink, {"memory", "register"});
  const std::string format = opt(a, "format", "json");
  member("format", format, {"json", "csv"});
  const std::string residency = opt(a, "residency", "device");
  member("residency", residency, {"device", "host", "file"});
  // file residency: each repetition is one mp_keyfile_merge (key files in,
  // key file out, ingest overlapped with the merge); the output file is
  // read back and verified like every other row
  const std::string fout = residency == "file" ? opt(a, "merged-out", fa + ".merged") : std::string();
  if (residency == "file" && (variant != "regular" || sink != "memory"))
    throw std::invalid_argument("--residency file takes the regular variant and the memory sink");
  // host residency: page-lock the tool's vectors before timing (pinned) or
  // leave them pageable -- what a plain std::vector caller passes; the
  // library then stages the chunks through pinned slots
  const std::string host_memory = opt(a, "host-memory", "pinned");
  member("host-memory", host_memory, {"pinned", "pageable"});
  const std::size_t reps = reps_of(a, 5);
  auto threads = a.kv.count("threads") ? to_list("threads", a.kv.at("threads"))
                                       : thread_sweep();
  std::vector<std::size_t> caches;
  const auto A = load_sorted(fa, "merge A");
  const auto B = load_sorted(fb, "merge B");
  const int dev = device_of(a);
  const mergepath::merge_input<std::int64_t> in{A, B};
  const std::size_t n = A.size() + B.size();
  std::vector<std::int64_t> ref(n);
  std::merge(A.begin(), A.end(), B.begin(), B.end(), ref.begin());
  const std::uint64_t ref_sum =
      mergepath::checksum_of(std::span<const std::int64_t>(ref));
  if (variant == "segmented") {
    if (a.kv.count("cache-elems"))
      caches = to_list("cache-elems", a.kv.at("cache-elems"));
    else
      for (std::size_t seg : {2, 5, 10})
        caches.push_back(std::max<std::size_t>(3, 3 * n / seg));
  } else {
    caches.push_back(0);
  }

  // device residency: the key files streamed into HBM once
  std::unique_ptr<DevBuf> dA, dB, dO;
  std::unique_ptr<Stream> st;
  if (residency == "device") {
    st = std::make_unique<Stream>();
    dA = std::make_unique<DevBuf>(A.size() * 8);
    dB = std::make_unique<DevBuf>(B.size() * 8);
    dO = std::make_unique<DevBuf>(n * 8);
    std::uint64_t got = 0;
    check_status(mp_keyfile_load(fa.c_str(), dA->p, A.size(), &got, dev, st->s));
    check_status(mp_keyfile_load(fb.c_str(), dB->p, B.size(), &got, dev, st->s));
  }

  std::vector<Row> rows;
  std::vector<std::int64_t> out(n);
  std::unique_ptr<PinScope> pa, pb, po;
  if (residency == "host" && host_memory == "pinned") {
    pa = std::make_unique<PinScope>(const_cast<std::int64_t *>(A.data()), A.size() * 8);
    pb = std::make_unique<PinScope>(const_cast<std::int64_t *>(B.data()), B.size() * 8);
    po = std::make_unique<PinScope>(out.data(), out.size() * 8);
  }
  for (std::size_t cache : caches) {
    for (std::size_t p : threads) {
      if (p == 0)
        throw std::invalid_argument("merge: thread counts must be positive");
      if (variant == "segmented" && cache < 3)
        throw std::invalid_argument("cache_elems must be >= 3");
      Row row;
      row.op = "merge";
      row.variant = variant;
      row.n = n;
      row.p = p;
      row.cache_elems = cache;
      row.reps = reps;
      mergepath::merge_stats stats;
      std::vector<double> times;
      for (std::size_t rep = 0; rep < reps; ++rep) {
        bool ok;
        if (residency == "device") {
          if (sink == "register") {
            std::uint64_t sum = 0;  // *sum is a device word (mergepath_b200.h)
            times.push_back(st->time([&] {
              check_status(mp_merge_checksum(MP_KEY_I64, dA->p, A.size(), dB->p,
                                             B.size(), static_cast<std::uint64_t *>(dO->p),
                                             st->s));
            }));
            check_cuda(cudaMemcpy(&sum, dO->p, 8, cudaMemcpyDeviceToHost), "D2H");
            ok = sum == ref_sum;
          } else {
            times.push_back(st->time([&] {
              check_status(mp_merge(MP_KEY_I64, dA->p, nullptr, A.size(), dB->p,
                                    nullptr, B.size(), dO->p, nullptr, st->s));
            }));
            check_cuda(cudaMemcpy(out.data(), dO->p, n * 8, cudaMemcpyDeviceToHost),
                       "D2H");
            ok = out == ref;
          }
        } else if (residency == "file") {
          std::uint64_t wrote = 0;
          times.push_back(wall([&] {
            check_status(mp_keyfile_merge(fa.c_str(), fb.c_str(), fout.c_str(), &wrote, dev));
          }));
          std::uint64_t got = 0;
          check_status(mp_keyfile_read(fout.c_str(), out.data(), out.size(), &got));
          ok = wrote == n && got == n && out == ref;
        } else if (sink == "register") {
          std::uint64_t sum = 0;
          times.push_back(wall([&] {
            sum = variant == "segmented"
                      ? mergepath::segmented_parallel_merge_checksum(in, p, cache)
                      : mergepath::parallel_merge_checksum(in, p);
          }));
          ok = sum == ref_sum;
        } else {
          times.push_back(wall([&] {
            if (variant == "segmented")
              mergepath::segmented_parallel_merge_into(in, std::span<std::int64_t>(out),
                                                       p, cache);
            else
              mergepath::parallel_merge_into(in, std::span<std::int64_t>(out), p);
          }));
          ok = out == ref;
        }
        if (!ok)
          throw mismatch_error("merge output diverged from the sequential reference");
      }
      // the reference's per-rep statistics (device replays of its searches)
      if (variant == "segmented")
        mergepath::detail::segmented_stats<std::int64_t, std::less<std::int64_t>>(
            in, p, cache, &stats);
      else
        mergepath::detail::regular_stats<std::int64_t, std::less<std::int64_t>>(
            in, p, &stats);
      row.partition_comparisons = stats.partition_comparisons;
      row.merge_steps = stats.merge_steps;
      const TimeStats ts = time_stats(times);
      row.median_seconds = ts.median;
      row.mean_seconds = ts.mean;
      row.verified = true;
      rows.push_back(row);
    }
  }
  fill_speedups(rows);
  Json meta = Json::object();
  meta.set("tool", Json::string("mergebench_b200"));
  meta.set("op", Json::string("merge"));
  meta.set("na", Json::integer(static_cast<long long>(A.size())));
  meta.set("nb", Json::integer(static_cast<long long>(B.size())));
  meta.set("sink", Json::string(sink));
  meta.set("hardware_threads", Json::integer(static_cast<long long>(host_threads())));
  meta.set("backend", Json::string("b200"));
  meta.set("device", Json::string(device_name(dev)));
  meta.set("residency", Json::string(residency));
  meta.set("host_memory", Json::string(residency == "host" ? host_memory : "n/a"));
  Json report = Json::object();
  report.set("meta", meta);
  Json arr = Json::array();
  for (const Row &r : rows)
    arr.a.push_back(row_json(r));
  report.set("rows", arr);
  emit(report, format, opt(a, "out", ""));
  return 0;
}

// ----------------------------------------------------------------- sort ---
int run_sort(const Args &a) {
  const std::string fin = need(a, "in");
  const std::string variant = opt(a, "variant", "plain");
  member("variant", variant, {"plain", "cache_efficient"});
  const std::string format = opt(a, "format", "json");
  member("format", format, {"json", "csv"});
  const std::string residency = opt(a, "residency", "device");
  member("residency", residency, {"device", "host", "file"});
  // file residency: each repetition is one mp_keyfile_sort (key file in,
  // sorted key file out), read back and verified
  const std::string fout = residency == "file" ? opt(a, "sorted-out", fin + ".sorted") : std::string();
  // host residency: page-lock the tool's vectors before timing (pinned) or
  // leave them pageable -- what a plain std::vector caller passes; the
  // library then stages the chunks through pinned slots
  const std::string host_memory = opt(a, "host-memory", "pinned");
  member("host-memory", host_memory, {"pinned", "pageable"});
  const std::size_t reps = reps_of(a, 3);
  const std::size_t cache = static_cast<std::size_t>(
      to_u64("cache-elems", opt(a, "cache-elems", std::to_string(3 * 4096))));
  auto threads = a.kv.count("threads") ? to_list("threads", a.kv.at("threads"))
                                       : thread_sweep();
  const auto data = read_keys(fin);
  const int dev = device_of(a);
  std::vector<std::int64_t> ref = data;
  std::sort(ref.begin(), ref.end());
  const std::size_t n = data.size();

  std::unique_ptr<DevBuf> dIn, dOut, dScr;
  std::unique_ptr<Stream> st;
  std::uint64_t scr_bytes = 0;
  if (residency == "device") {
    st = std::make_unique<Stream>();
    dIn = std::make_unique<DevBuf>(n * 8);
    dOut = std::make_unique<DevBuf>(n * 8);
    scr_bytes = mp_sort_scratch_bytes(MP_KEY_I64, 0, n);
    dScr = std::make_unique<DevBuf>(scr_bytes);
    std::uint64_t got = 0;
    check_status(mp_keyfile_load(fin.c_str(), dIn->p, n, &got, dev, st->s));
  }
  std::vector<Row> rows;
  std::unique_ptr<PinScope> pin_in;
  if (residency == "host" && host_memory == "pinned")
    pin_in = std::make_unique<PinScope>(const_cast<std::int64_t *>(data.data()), n * 8);
  for (std::size_t p : threads) {
    if (p == 0)
      throw std::invalid_argument("sort: thread counts must be positive");
    if (variant == "cache_efficient" && cache < 3)
      throw std::invalid_argument("cache_elems must be >= 3");
    Row row;
    row.op = "sort";
    row.variant = variant;
    row.n = n;
    row.p = p;
    row.cache_elems = variant == "cache_efficient" ? cache : 0;
    row.reps = reps;
    std::vector<double> times;
    std::vector<std::int64_t> out;
    for (std::size_t rep = 0; rep < reps; ++rep) {
      if (residency == "device") {
        times.push_back(st->time([&] {
          check_status(mp_sort_to(MP_KEY_I64, dIn->p, nullptr, dOut->p, nullptr, n,
                                  dScr->p, scr_bytes, st->s));
        }));
        out.resize(n);
        check_cuda(cudaMemcpy(out.data(), dOut->p, n * 8, cudaMemcpyDeviceToHost), "D2H");
      } else if (residency == "file") {
        std::uint64_t wrote = 0, got = 0;
        times.push_back(wall([&] {
          check_status(mp_keyfile_sort(fin.c_str(), fout.c_str(), &wrote, dev));
        }));
        out.assign(n, 0);
        check_status(mp_keyfile_read(fout.c_str(), out.data(), n, &got));
        if (wrote != n || got != n)
          throw mismatch_error("sorted key file has the wrong length");
      } else {
        times.push_back(wall([&] {
          out = variant == "cache_efficient"
                    ? mergepath::cache_efficient_parallel_sort(
                          std::span<const std::int64_t>(data), p, cache)
                    : mergepath::parallel_merge_sort(std::span<const std::int64_t>(data), p);
        }));
      }
      if (out != ref)
        throw mismatch_error("sort output diverged from the reference");
    }
    row.merge_rounds =
        mergepath::make_sort_plan(variant == "cache_efficient"
                                      ? mergepath::sort_variant::cache_efficient
                                      : mergepath::sort_variant::plain,
                                  n, variant == "cache_efficient" ? cache : 0)
            .tree_levels;
    const TimeStats ts = time_stats(times);
    row.median_seconds = ts.median;
    row.mean_seconds = ts.mean;
    row.verified = true;
    rows.push_back(row);
  }
  fill_speedups(rows);
  Json meta = Json::object();
  meta.set("tool", Json::string("mergebench_b200"));
  meta.set("op", Json::string("sort"));
  meta.set("n", Json::integer(static_cast<long long>(n)));
  meta.set("variant", Json::string(variant));
  meta.set("hardware_threads", Json::integer(static_cast<long long>(host_threads())));
  meta.set("backend", Json::string("b200"));
  meta.set("device", Json::string(device_name(dev)));
  meta.set("residency", Json::string(residency));
  meta.set("host_memory", Json::string(residency == "host" ? host_memory : "n/a"));
  Json report = Json::object();
  report.set("meta", meta);
  Json arr = Json::array();
  for (const Row &r : rows)
    arr.a.push_back(row_json(r));
  report.set("rows", arr);
  emit(report, format, opt(a, "out", ""));
  return 0;
}

// --------------------------------------------------------------- report ---
int run_report(const Args &a) {
  const std::string fin = need(a, "in");
  const std::string format = opt(a, "format", "csv");
  member("format", format, {"json", "csv"});
  std::ifstream in(fin);
  if (!in)
    throw io_error("cannot open: " + fin);
  std::stringstream ss;
  ss << in.rdbuf();
  const Json report = parse_json(ss.str());
  const Json *rows = report.kind == Json::Obj ? report.get("rows") : nullptr;
  if (!rows || rows->kind != Json::Arr)
    throw std::invalid_argument("report file has no rows");
  emit(report, format, opt(a, "out", ""));
  return 0;
}

void usage(std::ostream &out) {
  out << "usage: mergebench_b200 {gen|merge|sort|report} [options]\n"
         "  gen    --dist uniform|all_equal|disjoint_ranges|interleaved --na N --nb N\n"
         "         [--seed S] --out-a F --out-b F [--format bin|text]\n"
         "  merge  --a F --b F [--variant regular|segmented] [--threads P,..]\n"
         "         [--cache-elems C,..] [--reps R>=3] [--sink memory|register]\n"
         "         [--format json|csv] [--out F] [--residency device|host] [--host-memory pinned|pageable] [--device N]\n"
         "  sort   --in F [--variant plain|cache_efficient] [--threads P,..]\n"
         "         [--cache-elems C] [--reps R>=3] [--format json|csv] [--out F]\n"
         "         [--residency device|host] [--host-memory pinned|pageable] [--device N]\n"
         "  report --in F [--format json|csv] [--out F]\n";
}

}  // namespace

int main(int argc, char **argv) {
  if (argc < 2) {
    usage(std::cerr);
    return 1;
  }
  const std::string cmd = argv[1];
  if (cmd == "-h" || cmd == "--help") {
    usage(std::cout);
    return 0;
  }
  try {
    if (cmd == "gen")
      return run_gen(parse_args(argc, argv, 2,
                                {"dist", "na", "nb", "seed", "out-a", "out-b", "format"}));
    if (cmd == "merge")
      return run_merge(parse_args(argc, argv, 2,
                                  {"a", "b", "variant", "threads", "cache-elems", "reps",
                                   "sink", "format", "out", "residency", "host-memory", "device", "merged-out"}));
    if (cmd == "sort")
      return run_sort(parse_args(argc, argv, 2,
                                 {"in", "variant", "threads", "cache-elems", "reps",
                                  "format", "out", "residency", "host-memory", "device", "sorted-out"}));
    if (cmd == "report")
      return run_report(parse_args(argc, argv, 2, {"in", "format", "out"}));
    if (cmd == "cachesim")
      throw usage_error("cachesim (CPU cache model) is not part of the B200 backend");
    throw usage_error("unknown subcommand: " + cmd);
  } catch (const usage_error &e) {
    std::cerr << "error: " << e.what() << '\n';
    usage(std::cerr);
    return 1;
  } catch (const mismatch_error &e) {
    std::cerr << "error: " << e.what() << '\n';
    return 4;
  } catch (const std::invalid_argument &e) {
    std::cerr << "error: " << e.what() << '\n';
    return 3;
  } catch (const std::exception &e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  }
}
