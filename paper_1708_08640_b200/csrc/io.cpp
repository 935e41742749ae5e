// io.cpp -- the reference's text formats and host-side data preparation
// (SURVEY.md 8(f) rows 1-2), native C++ in the same library:
//
//   * COO text parse  (parse_coo_file / infer_dims, src/sparse_data.cpp:66-233):
//     the file is mapped once, the header is resolved from its first two data
//     lines exactly as the reference does, then the entry lines are parsed by
//     all host threads in line-aligned chunks; the first error in file order
//     is reported with the reference's ParseError text and line number.  The
//     checks of the SparseTensor / CoupledMatrix constructors (check_entries:
//     range, finiteness, duplicate tuples) run on the device
//     (cmtf_gpu_check_entries, context.cu).
//   * COO text write  (write_coo, src/sparse_data.cpp:279-302): %.17g values,
//     formatted by all threads, written in order.
//   * split_train_test (src/sparse_data.cpp:311-342): the reference's
//     Fisher-Yates over entry ids with the Split stream (inherently serial:
//     the same draws give the same split), gathers in parallel.
//   * save_model / load_model (src/model_io.cpp:94-179): CORE / FACTOR n /
//     COUPLED c sections, 17 significant digits.
//
// Error codes: CMTF_EPARSE (ParseError), CMTF_EVALIDATION (ValidationError).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cmtf_b200.h"
#include "host_rng.hpp"

namespace cmtfb {
int io_fail(int code, const std::string& msg);  // context.cu: sets the last error
}

using cmtfb::io_fail;

struct cmtf_coo {
  int32_t order = 0;
  std::vector<uint32_t> header;  // empty when absent
  std::vector<uint32_t> dims;
  std::vector<uint32_t> idx;     // 0-based, AoS
  std::vector<double> vals;
};

struct cmtf_model_file {
  std::vector<uint32_t> ranks;
  std::vector<double> core;
  std::vector<uint32_t> frows, fcols;
  std::vector<std::vector<double>> factors;
  std::vector<int32_t> cmode;
  std::vector<uint32_t> crows, ccols;
  std::vector<std::vector<double>> couplings;
};

namespace {

int n_threads(int32_t requested) {
  if (requested > 0) return requested;
  const unsigned hc = std::thread::hardware_concurrency();
  return hc ? (int)hc : 1;
}

template <class F>
void parallel_for(int T, F&& f) {
  if (T <= 1) {
    f(0);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T - 1);
  for (int t = 1; t < T; ++t) th.emplace_back([&f, t] { f(t); });
  f(0);
  for (auto& x : th) x.join();
}

// std::istringstream >> std::string separators in the "C" locale
inline bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

struct Tok {
  const char* p;
  size_t n;
  std::string str() const { return std::string(p, n); }
};

// One line [b, e) (no '\n'): trailing '\r' dropped, '#' comment stripped,
// whitespace tokens (src/sparse_data.cpp:188-192, 83-89).
inline void tokenize(const char* b, const char* e, std::vector<Tok>& out) {
  out.clear();
  if (e <= b) return;
  if (e[-1] == '\r') --e;
  const void* h = std::memchr(b, '#', (size_t)(e - b));
  if (h) e = static_cast<const char*>(h);
  const char* p = b;
  while (p < e) {
    while (p < e && is_space(*p)) ++p;
    if (p >= e) break;
    const char* q = p;
    while (q < e && !is_space(*q)) ++q;
    out.push_back({p, (size_t)(q - p)});
    p = q;
  }
}

// is_integer_token (src/sparse_data.cpp:73-81)
bool is_integer_token(const Tok& t) {
  if (t.n == 0) return false;
  size_t i = t.p[0] == '+' ? 1 : 0;
  if (i == t.n) return false;
  for (; i < t.n; ++i)
    if (t.p[i] < '0' || t.p[i] > '9') return false;
  return true;
}

struct LineError {
  bool set = false;
  uint64_t line = 0;  // chunk-local (0-based line within the chunk) until resolved
  std::string msg;     // without the " (line N)" suffix
};

// parse_index (src/sparse_data.cpp:91-102): from_chars into long long, >= 1,
// <= 2^32 - 1.  Returns false and fills `err` on failure.
inline bool parse_index(const Tok& t, uint32_t* out, std::string* err) {
  long long v = 0;
  auto [ptr, ec] = std::from_chars(t.p, t.p + t.n, v);
  if (ec != std::errc() || ptr != t.p + t.n) {
    *err = "expected an integer index, got '" + t.str() + "'";
    return false;
  }
  if (v < 1) {
    *err = "index must be >= 1";
    return false;
  }
  if (v > 0xffffffffLL) {
    *err = "index too large";
    return false;
  }
  *out = (uint32_t)v;
  return true;
}

// parse_value (src/sparse_data.cpp:104-119): std::stod semantics (strtod;
// ERANGE -> out_of_range -> "expected a numeric value"), whole token
// consumed, finite.
inline bool parse_value(const Tok& t, double* out, std::string* err) {
  char buf[128];
  std::string big;
  const char* s;
  if (t.n < sizeof buf) {
    std::memcpy(buf, t.p, t.n);
    buf[t.n] = 0;
    s = buf;
  } else {
    big = t.str();
    s = big.c_str();
  }
  char* end = nullptr;
  const int saved = errno;
  errno = 0;
  const double v = std::strtod(s, &end);
  const bool range = errno == ERANGE;
  errno = saved;
  if (end == s || range || (size_t)(end - s) != t.n) {
    *err = "expected a numeric value, got '" + t.str() + "'";
    return false;
  }
  if (!std::isfinite(v)) {
    *err = "value is not finite";
    return false;
  }
  *out = v;
  return true;
}

struct Chunk {
  const char* b;
  const char* e;
  uint64_t lines = 0;  // newline-terminated lines (+1 for a final unterminated line)
  std::vector<uint32_t> idx;
  std::vector<double> vals;
  LineError err;
};

// consume_entry (src/sparse_data.cpp:138-146) over the lines of a chunk
void parse_chunk(Chunk& c, size_t tpe) {
  std::vector<Tok> toks;
  const size_t order = tpe - 1;
  const char* p = c.b;
  uint64_t ln = 0;
  std::string err;
  while (p < c.e) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(c.e - p)));
    const char* le = nl ? nl : c.e;
    tokenize(p, le, toks);
    if (!toks.empty()) {
      if (toks.size() != tpe) {
        c.err = {true, ln,
                 "expected " + std::to_string(tpe) + " fields, got " + std::to_string(toks.size())};
        return;
      }
      uint32_t ix[64];
      for (size_t n = 0; n < order; ++n) {
        if (!parse_index(toks[n], &ix[n], &err)) {
          c.err = {true, ln, err};
          return;
        }
      }
      double v;
      if (!parse_value(toks[order], &v, &err)) {
        c.err = {true, ln, err};
        return;
      }
      for (size_t n = 0; n < order; ++n) c.idx.push_back(ix[n] - 1);
      c.vals.push_back(v);
    }
    ++ln;
    p = nl ? nl + 1 : c.e;
  }
  c.lines = ln;
}

struct Mapped {
  const char* data = nullptr;
  size_t size = 0;
  void* map = nullptr;
  ~Mapped() {
    if (map && map != MAP_FAILED) munmap(map, size);
  }
};

int map_file(const char* path, Mapped& m) {
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) return io_fail(CMTF_EPARSE, std::string("cannot open '") + path + "'");
  struct stat st {};
  if (fstat(fd, &st) != 0 || S_ISDIR(st.st_mode)) {
    ::close(fd);
    return io_fail(CMTF_EPARSE, std::string("cannot open '") + path + "'");
  }
  m.size = (size_t)st.st_size;
  if (m.size) {
    m.map = mmap(nullptr, m.size, PROT_READ, MAP_PRIVATE, fd, 0);
    if (m.map == MAP_FAILED) {
      ::close(fd);
      return io_fail(CMTF_EPARSE, std::string("cannot open '") + path + "'");
    }
    madvise(m.map, m.size, MADV_SEQUENTIAL | MADV_WILLNEED);
    m.data = static_cast<const char*>(m.map);
  }
  ::close(fd);
  return CMTF_OK;
}

std::string line_msg(const std::string& m, uint64_t line) {
  return m + " (line " + std::to_string(line) + ")";
}

}  // namespace

extern "C" {

int cmtf_coo_parse(const char* path, int32_t expected_order, int32_t threads, cmtf_coo** out) {
  if (!path || !out) return io_fail(CMTF_EVALIDATION, "null argument");
  *out = nullptr;
  Mapped m;
  if (int rc = map_file(path, m)) return rc;
  const char* const B = m.data;
  const char* const E = m.data + m.size;
  auto coo = std::make_unique<cmtf_coo>();
  std::string err;

  // ---- the first two data lines decide the header (resolve, :148-178) ----
  struct Pending {
    std::vector<Tok> toks;
    uint64_t line;        // 1-based
    const char* begin;    // start of the line
    const char* next;     // start of the following line
  };
  std::vector<Pending> pend;
  {
    const char* p = B;
    uint64_t ln = 0;
    std::vector<Tok> toks;
    while (p < E && pend.size() < 2) {
      const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(E - p)));
      const char* le = nl ? nl : E;
      ++ln;
      tokenize(p, le, toks);
      const char* nx = nl ? nl + 1 : E;
      if (!toks.empty()) pend.push_back({toks, ln, p, nx});
      p = nx;
    }
  }
  if (pend.empty())
    return io_fail(CMTF_EPARSE, std::string("'") + path + "' contains no data");
  const auto& first = pend[0];
  const bool first_all_int =
      std::all_of(first.toks.begin(), first.toks.end(), [](const Tok& t) { return is_integer_token(t); });
  bool header = false;
  if (pend.size() >= 2 && first.toks.size() + 1 == pend[1].toks.size() && first_all_int) {
    header = true;
  } else if (pend.size() == 1 && first_all_int &&
             (expected_order == 0 || (int)first.toks.size() == expected_order)) {
    header = true;  // header-only file: an empty tensor / matrix
  }
  size_t tpe;
  const char* start;
  uint64_t start_line;  // 1-based number of the line at `start`
  if (header) {
    for (const auto& t : first.toks) {
      uint32_t v;
      if (!parse_index(t, &v, &err)) return io_fail(CMTF_EPARSE, line_msg(err, first.line));
      coo->header.push_back(v);
    }
    tpe = first.toks.size() + 1;
    start = first.next;
    start_line = first.line + 1;
  } else {
    if (first.toks.size() < 2)
      return io_fail(CMTF_EPARSE, line_msg("entry line needs at least one index and a value",
                                           first.line));
    tpe = first.toks.size();
    start = first.begin;
    start_line = first.line;
  }
  if (tpe - 1 > 64) return io_fail(CMTF_EPARSE, std::string("'") + path + "': too many indices per entry");

  // ---- entry lines, in parallel line-aligned chunks ----
  const size_t rest = (size_t)(E - start);
  int T = n_threads(threads);
  if (rest < (size_t)(1 << 20)) T = 1;
  std::vector<Chunk> ch(T);
  {
    const char* b = start;
    for (int t = 0; t < T; ++t) {
      const char* e = t + 1 == T ? E : start + rest * (t + 1) / T;
      if (e < b) e = b;
      if (t + 1 < T && e < E) {  // extend to the end of the line
        const char* nl = static_cast<const char*>(std::memchr(e, '\n', (size_t)(E - e)));
        e = nl ? nl + 1 : E;
      }
      ch[t].b = b;
      ch[t].e = e;
      b = e;
    }
  }
  parallel_for(T, [&](int t) { parse_chunk(ch[t], tpe); });
  uint64_t line0 = start_line, total = 0;
  for (int t = 0; t < T; ++t) {
    if (ch[t].err.set) return io_fail(CMTF_EPARSE, line_msg(ch[t].err.msg, line0 + ch[t].err.line));
    line0 += ch[t].lines;
    total += ch[t].vals.size();
  }
  const size_t order = tpe - 1;
  if (expected_order != 0 && (int)order != expected_order)
    return io_fail(CMTF_EPARSE, std::string("'") + path + "': expected " +
                                    std::to_string(expected_order) + " indices per entry, found " +
                                    std::to_string(order));
  coo->order = (int32_t)order;
  coo->idx.resize(total * order);
  coo->vals.resize(total);
  std::vector<uint64_t> off(T + 1, 0);
  for (int t = 0; t < T; ++t) off[t + 1] = off[t] + ch[t].vals.size();
  parallel_for(T, [&](int t) {
    std::copy(ch[t].vals.begin(), ch[t].vals.end(), coo->vals.begin() + off[t]);
    std::copy(ch[t].idx.begin(), ch[t].idx.end(), coo->idx.begin() + off[t] * order);
    std::vector<uint32_t>().swap(ch[t].idx);
    std::vector<double>().swap(ch[t].vals);
  });
  // infer_dims (:217-227): the header, else the per-mode maximum index + 1
  if (!coo->header.empty()) {
    coo->dims = coo->header;
  } else {
    std::vector<std::vector<uint32_t>> mx(T, std::vector<uint32_t>(order, 0));
    parallel_for(T, [&](int t) {
      const uint64_t lo = total * t / T, hi = total * (t + 1) / T;
      for (uint64_t e = lo; e < hi; ++e)
        for (size_t n = 0; n < order; ++n)
          mx[t][n] = std::max(mx[t][n], coo->idx[e * order + n] + 1);
    });
    coo->dims.assign(order, 0);
    for (int t = 0; t < T; ++t)
      for (size_t n = 0; n < order; ++n) coo->dims[n] = std::max(coo->dims[n], mx[t][n]);
  }
  *out = coo.release();
  return CMTF_OK;
}

int32_t cmtf_coo_order(const cmtf_coo* c) { return c ? c->order : 0; }
uint64_t cmtf_coo_nnz(const cmtf_coo* c) { return c ? c->vals.size() : 0; }
int32_t cmtf_coo_has_header(const cmtf_coo* c) { return c && !c->header.empty(); }
const uint32_t* cmtf_coo_dims(const cmtf_coo* c) { return c ? c->dims.data() : nullptr; }
const uint32_t* cmtf_coo_indices(const cmtf_coo* c) { return c ? c->idx.data() : nullptr; }
const double* cmtf_coo_values(const cmtf_coo* c) { return c ? c->vals.data() : nullptr; }
void cmtf_coo_free(cmtf_coo* c) { delete c; }

int cmtf_coo_write(const char* path, int32_t order, const uint32_t* dims, const uint32_t* idx,
                   const double* vals, uint64_t nnz, int32_t threads) {
  if (!path || order < 1 || !dims) return io_fail(CMTF_EVALIDATION, "invalid arguments");
  FILE* f = std::fopen(path, "wb");
  if (!f) return io_fail(CMTF_EPARSE, std::string("cannot write '") + path + "'");
  std::string head;
  for (int n = 0; n < order; ++n) head += std::to_string(dims[n]) + (n + 1 < order ? " " : "\n");
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  // formatted in blocks by all threads, written in order
  const int T = n_threads(threads);
  const uint64_t block = 1u << 20;
  for (uint64_t b0 = 0; b0 < nnz && ok; b0 += block * T) {
    std::vector<std::string> buf(T);
    parallel_for(T, [&](int t) {
      const uint64_t lo = b0 + block * t, hi = std::min<uint64_t>(nnz, lo + block);
      std::string& s = buf[t];
      if (lo >= hi) return;
      s.reserve((hi - lo) * (12 * order + 26));
      char num[64];
      for (uint64_t e = lo; e < hi; ++e) {
        for (int n = 0; n < order; ++n) {
          auto r = std::to_chars(num, num + sizeof num, (unsigned long long)idx[e * order + n] + 1);
          s.append(num, r.ptr);
          s.push_back(' ');
        }
        const int k = std::snprintf(num, sizeof num, "%.17g", vals[e]);
        s.append(num, (size_t)k);
        s.push_back('\n');
      }
    });
    for (int t = 0; t < T && ok; ++t)
      ok = std::fwrite(buf[t].data(), 1, buf[t].size(), f) == buf[t].size();
  }
  if (std::fclose(f) != 0) ok = false;
  if (!ok) return io_fail(CMTF_EPARSE, std::string("write failed for '") + path + "'");
  return CMTF_OK;
}

int cmtf_split_train_test(int32_t order, const uint32_t* idx, const double* vals, uint64_t nnz,
                          double test_fraction, uint64_t seed, uint32_t* train_idx,
                          double* train_vals, uint32_t* test_idx, double* test_vals,
                          uint64_t* n_test_out, int32_t threads) {
  if (nnz == 0) return io_fail(CMTF_EVALIDATION, "cannot split an empty tensor");
  if (!(test_fraction > 0.0) || !(test_fraction < 1.0))
    return io_fail(CMTF_EVALIDATION, "test fraction must be in (0, 1)");
  const uint64_t n_test = (uint64_t)std::llround(test_fraction * (double)nnz);
  if (n_test_out) *n_test_out = n_test;
  if (!train_idx && !test_idx) return CMTF_OK;  // size query
  // Fisher-Yates over the entry ids with the Split stream (:322-326)
  auto rng = cmtfb::make_rng(seed, cmtfb::kStreamSplit, 0);
  std::vector<uint64_t> ids64;
  std::vector<uint32_t> ids32;
  const bool narrow = nnz <= 0xffffffffull;
  if (narrow) {
    ids32.resize(nnz);
    std::iota(ids32.begin(), ids32.end(), 0u);
    for (uint64_t i = nnz - 1; i > 0; --i) std::swap(ids32[i], ids32[cmtfb::bounded(rng, i + 1)]);
  } else {
    ids64.resize(nnz);
    std::iota(ids64.begin(), ids64.end(), uint64_t{0});
    for (uint64_t i = nnz - 1; i > 0; --i) std::swap(ids64[i], ids64[cmtfb::bounded(rng, i + 1)]);
  }
  auto id = [&](uint64_t i) -> uint64_t { return narrow ? ids32[i] : ids64[i]; };
  // test = first n_test shuffled ids, train = the rest, both in shuffled order
  const int T = n_threads(threads);
  parallel_for(T, [&](int t) {
    const uint64_t lo = nnz * t / T, hi = nnz * (t + 1) / T;
    for (uint64_t i = lo; i < hi; ++i) {
      const uint64_t e = id(i);
      uint32_t* di;
      double* dv;
      uint64_t k;
      if (i < n_test) {
        di = test_idx;
        dv = test_vals;
        k = i;
      } else {
        di = train_idx;
        dv = train_vals;
        k = i - n_test;
      }
      if (!di) continue;
      for (int n = 0; n < order; ++n) di[k * order + n] = idx[e * order + n];
      dv[k] = vals[e];
    }
  });
  return CMTF_OK;
}

// ---- model text format (src/model_io.cpp) ----

namespace {

// write_values (:15-23): per_line values per line, "%.17g"
void write_values(std::string& s, const double* v, size_t n, size_t per_line) {
  char buf[64];
  for (size_t i = 0; i < n; ++i) {
    const int k = std::snprintf(buf, sizeof buf, "%.17g", v[i]);
    s.append(buf, (size_t)k);
    s.push_back((i + 1) % per_line == 0 ? '\n' : ' ');
  }
  if (n % per_line != 0) s.push_back('\n');
}

// validate_model (src/tucker.cpp:208-224)
int validate_model(int32_t order, const uint32_t* ranks, const uint32_t* fcols, int32_t nf,
                   int32_t nc, const int32_t* cmode, const uint32_t* ccols) {
  if (nf != order)
    return io_fail(CMTF_EVALIDATION, "model has " + std::to_string(nf) +
                                         " factors for a core of order " + std::to_string(order));
  for (int n = 0; n < nf; ++n)
    if (fcols[n] != ranks[n])
      return io_fail(CMTF_EVALIDATION, "factor " + std::to_string(n + 1) + " width does not match rank");
  for (int c = 0; c < nc; ++c) {
    if (cmode[c] < 0 || cmode[c] >= order)
      return io_fail(CMTF_EVALIDATION, "coupling mode out of range");
    if (ccols[c] != ranks[cmode[c]])
      return io_fail(CMTF_EVALIDATION, "coupled factor width does not match rank");
  }
  return CMTF_OK;
}

}  // namespace

int cmtf_model_save(const char* path, int32_t order, const uint32_t* ranks, int32_t cp,
                    const double* core, const uint32_t* factor_rows,
                    const double* const* factors, int32_t n_coupled, const int32_t* coupled_modes,
                    const uint32_t* coupled_rows, const double* const* couplings) {
  if (!path || order < 1 || !ranks || !core) return io_fail(CMTF_EVALIDATION, "invalid arguments");
  {
    std::vector<uint32_t> ccols(n_coupled);
    for (int c = 0; c < n_coupled; ++c)
      ccols[c] = (coupled_modes[c] >= 0 && coupled_modes[c] < order) ? ranks[coupled_modes[c]] : 0;
    if (int rc = validate_model(order, ranks, ranks, order, n_coupled, coupled_modes, ccols.data()))
      return rc;
  }
  std::string s = "CORE\n";
  for (int n = 0; n < order; ++n) s += std::to_string(ranks[n]) + (n + 1 < order ? " " : "\n");
  size_t dense = 1;
  for (int n = 0; n < order; ++n) dense *= ranks[n];
  if (cp) {
    // CP cores are written densely (:105-112): the superdiagonal at k * sum(strides)
    std::vector<double> d(dense, 0.0);
    size_t step = 0, stride = 1;
    for (int n = order - 1; n >= 0; --n) {
      step += stride;
      stride *= ranks[n];
    }
    for (uint32_t k = 0; k < ranks[0]; ++k) d[k * step] = core[k];
    write_values(s, d.data(), dense, ranks[order - 1]);
  } else {
    write_values(s, core, dense, ranks[order - 1]);
  }
  for (int n = 0; n < order; ++n) {
    s += "FACTOR " + std::to_string(n + 1) + "\n" + std::to_string(factor_rows[n]) + " " +
         std::to_string(ranks[n]) + "\n";
    write_values(s, factors[n], (size_t)factor_rows[n] * ranks[n], ranks[n]);
  }
  for (int c = 0; c < n_coupled; ++c) {
    const uint32_t J = ranks[coupled_modes[c]];
    s += "COUPLED " + std::to_string(coupled_modes[c] + 1) + "\n" +
         std::to_string(coupled_rows[c]) + " " + std::to_string(J) + "\n";
    write_values(s, couplings[c], (size_t)coupled_rows[c] * J, J);
  }
  FILE* f = std::fopen(path, "wb");
  if (!f) return io_fail(CMTF_EPARSE, std::string("cannot write '") + path + "'");
  const bool ok = std::fwrite(s.data(), 1, s.size(), f) == s.size();
  if (std::fclose(f) != 0 || !ok)
    return io_fail(CMTF_EPARSE, std::string("write failed for '") + path + "'");
  return CMTF_OK;
}

namespace {

// Reader (:27-72): section headers and shape lines are whole lines, value
// blocks are free-form token runs
struct ModelReader {
  const char* p;
  const char* e;
  std::vector<Tok> line;
  size_t pos = 0;

  bool raw_line(std::vector<Tok>& toks) {
    if (p >= e) return false;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(e - p)));
    const char* le = nl ? nl : e;
    // no comment stripping in the model format: tokenize on whitespace only
    toks.clear();
    const char* q = p;
    const char* end = (le > p && le[-1] == '\r') ? le - 1 : le;
    while (q < end) {
      while (q < end && is_space(*q)) ++q;
      if (q >= end) break;
      const char* r = q;
      while (r < end && !is_space(*r)) ++r;
      toks.push_back({q, (size_t)(r - q)});
      q = r;
    }
    p = nl ? nl + 1 : e;
    return true;
  }
  // tokens of the next non-blank line; empty at end of file
  int next_line(std::vector<Tok>& out) {
    if (pos < line.size())
      return io_fail(CMTF_EPARSE, "model file: unexpected extra tokens before '" +
                                      line[pos].str() + "'");
    while (raw_line(line)) {
      pos = line.size();
      if (!line.empty()) {
        out = line;
        return CMTF_OK;
      }
    }
    out.clear();
    return CMTF_OK;
  }
  int next_value(double* v) {
    while (pos >= line.size()) {
      if (!raw_line(line)) return io_fail(CMTF_EPARSE, "model file ends inside a value block");
      pos = 0;
    }
    const Tok& t = line[pos++];
    char buf[128];
    std::string big;
    const char* s;
    if (t.n < sizeof buf) {
      std::memcpy(buf, t.p, t.n);
      buf[t.n] = 0;
      s = buf;
    } else {
      big = t.str();
      s = big.c_str();
    }
    char* end = nullptr;
    const int saved = errno;
    errno = 0;
    *v = std::strtod(s, &end);
    const bool range = errno == ERANGE;
    errno = saved;
    if (end == s || range || (size_t)(end - s) != t.n)
      return io_fail(CMTF_EPARSE, "model file: expected a number, got '" + t.str() + "'");
    return CMTF_OK;
  }
};

// to_u32 (:74-84): std::stoul semantics (strtoul: leading blanks and a sign
// accepted, trailing characters ignored, ERANGE rejected), then 1 .. 2^32-1
int to_u32(const Tok& t, uint32_t* out) {
  const std::string s = t.str();
  char* end = nullptr;
  const int saved = errno;
  errno = 0;
  const unsigned long v = std::strtoul(s.c_str(), &end, 10);
  const bool bad = end == s.c_str() || errno == ERANGE;
  errno = saved;
  if (bad || v == 0 || v > 0xffffffffUL)
    return io_fail(CMTF_EPARSE, "model file: expected a positive integer, got '" + s + "'");
  *out = (uint32_t)v;
  return CMTF_OK;
}

}  // namespace

int cmtf_model_load(const char* path, cmtf_model_file** out) {
  if (!path || !out) return io_fail(CMTF_EVALIDATION, "null argument");
  *out = nullptr;
  Mapped m;
  if (int rc = map_file(path, m)) return rc;
  ModelReader rd{m.data, m.data + m.size};
  auto mf = std::make_unique<cmtf_model_file>();
  std::vector<Tok> l;
  if (int rc = rd.next_line(l)) return rc;
  if (l.size() != 1 || l[0].str() != "CORE")
    return io_fail(CMTF_EPARSE, "model file must start with a CORE section");
  if (int rc = rd.next_line(l)) return rc;
  for (const auto& t : l) {
    uint32_t v;
    if (int rc = to_u32(t, &v)) return rc;
    mf->ranks.push_back(v);
  }
  if (mf->ranks.empty()) return io_fail(CMTF_EPARSE, "model file: missing ranks line");
  size_t cs = 1;
  for (auto j : mf->ranks) cs *= j;
  mf->core.resize(cs);
  for (double& v : mf->core)
    if (int rc = rd.next_value(&v)) return rc;
  for (;;) {
    if (int rc = rd.next_line(l)) return rc;
    if (l.empty()) break;
    if (l.size() != 2) return io_fail(CMTF_EPARSE, "model file: malformed section header");
    const std::string kind = l[0].str();
    const bool is_factor = kind == "FACTOR", is_coupled = kind == "COUPLED";
    if (!is_factor && !is_coupled)
      return io_fail(CMTF_EPARSE, "model file: unknown section '" + kind + "'");
    uint32_t tag;
    if (int rc = to_u32(l[1], &tag)) return rc;
    if (int rc = rd.next_line(l)) return rc;
    if (l.size() != 2) return io_fail(CMTF_EPARSE, "model file: section needs a 'rows cols' line");
    uint32_t rows, cols;
    if (int rc = to_u32(l[0], &rows)) return rc;
    if (int rc = to_u32(l[1], &cols)) return rc;
    std::vector<double> vals((size_t)rows * cols);
    for (double& v : vals)
      if (int rc = rd.next_value(&v)) return rc;
    if (is_factor) {
      if (tag != mf->factors.size() + 1)
        return io_fail(CMTF_EPARSE, "model file: FACTOR sections must appear in order");
      mf->frows.push_back(rows);
      mf->fcols.push_back(cols);
      mf->factors.push_back(std::move(vals));
    } else {
      mf->cmode.push_back((int32_t)tag - 1);
      mf->crows.push_back(rows);
      mf->ccols.push_back(cols);
      mf->couplings.push_back(std::move(vals));
    }
  }
  if (int rc = validate_model((int32_t)mf->ranks.size(), mf->ranks.data(), mf->fcols.data(),
                              (int32_t)mf->factors.size(), (int32_t)mf->couplings.size(),
                              mf->cmode.data(), mf->ccols.data()))
    return rc;
  *out = mf.release();
  return CMTF_OK;
}

int32_t cmtf_model_order(const cmtf_model_file* m) { return m ? (int32_t)m->ranks.size() : 0; }
const uint32_t* cmtf_model_ranks(const cmtf_model_file* m) { return m ? m->ranks.data() : nullptr; }
const double* cmtf_model_core(const cmtf_model_file* m) { return m ? m->core.data() : nullptr; }
uint32_t cmtf_model_factor_rows(const cmtf_model_file* m, int32_t n) {
  return m && n >= 0 && n < (int32_t)m->frows.size() ? m->frows[n] : 0;
}
const double* cmtf_model_factor(const cmtf_model_file* m, int32_t n) {
  return m && n >= 0 && n < (int32_t)m->factors.size() ? m->factors[n].data() : nullptr;
}
int32_t cmtf_model_n_coupled(const cmtf_model_file* m) {
  return m ? (int32_t)m->couplings.size() : 0;
}
int32_t cmtf_model_coupled_mode(const cmtf_model_file* m, int32_t c) {
  return m && c >= 0 && c < (int32_t)m->cmode.size() ? m->cmode[c] : -1;
}
uint32_t cmtf_model_coupled_rows(const cmtf_model_file* m, int32_t c) {
  return m && c >= 0 && c < (int32_t)m->crows.size() ? m->crows[c] : 0;
}
const double* cmtf_model_coupled(const cmtf_model_file* m, int32_t c) {
  return m && c >= 0 && c < (int32_t)m->couplings.size() ? m->couplings[c].data() : nullptr;
}
void cmtf_model_free(cmtf_model_file* m) { delete m; }

}  // extern "C"
