// FROSTT text ingestion: parallel host parse straight into (pinned) staging
// buffers; the canonicalisation that follows runs on the GPU.
//
// Restates parse_frostt (pkg/src/alto/tensor.py:245-296): one-based indices
// then a value per line, `#` comments and blank lines skipped, the mode count
// fixed by the first data line, and the same error classes with the line
// number of the first offending line in file order:
//   "expected at least one index and a value", "expected F fields, got G",
//   "bad index in [...]", "indices are one-based, got [...]",
//   "bad value '...'", "non-finite value '...'".
// Integers accept an optional sign and decimal digits; values are parsed with
// strtod (correctly rounded, like Python's float) after rejecting the forms
// Python's float() rejects (hex, "nan(...)"). Python's digit-group
// underscores are not accepted.
#include <ctype.h>
#include <errno.h>
#include <limits.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "alto_common.cuh"

namespace alto {
namespace {

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// next token in [p, e): returns false at end of line
inline bool next_token(const char *&p, const char *e, const char *&tb, const char *&te) {
  while (p < e && is_space(*p)) ++p;
  if (p >= e) return false;
  tb = p;
  while (p < e && !is_space(*p)) ++p;
  te = p;
  return true;
}

inline bool data_line(const char *b, const char *e, int *fields) {
  const char *p = b;
  while (p < e && is_space(*p)) ++p;
  if (p >= e || *p == '#') return false;
  int n = 0;
  const char *tb, *te;
  while (next_token(p, e, tb, te)) ++n;
  *fields = n;
  return true;
}

inline bool parse_int(const char *b, const char *e, long long *out) {
  const char *p = b;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  if (p >= e) return false;
  long long v = 0;
  for (; p < e; ++p) {
    if (*p < '0' || *p > '9') return false;
    const int d = *p - '0';
    if (v > (LLONG_MAX - d) / 10) return false;
    v = v * 10 + d;
  }
  *out = neg ? -v : v;
  return true;
}

inline bool parse_value(const char *b, const char *e, double *out) {
  char buf[128];
  const size_t n = (size_t)(e - b);
  if (n == 0 || n >= sizeof buf) return false;
  for (const char *p = b; p < e; ++p)
    if (*p == 'x' || *p == 'X' || *p == '(' || *p == 'p' || *p == 'P') return false;
  memcpy(buf, b, n);
  buf[n] = 0;
  char *end = nullptr;
  errno = 0;
  const double v = strtod(buf, &end);
  if (end != buf + n) return false;
  *out = v;  // overflow gives +-inf like Python's float("1e999")
  return true;
}

std::string int_list(const long long *v, int count) {
  // "[1, 2, 3]" as Python prints a list of ints
  std::string s = "[";
  for (int i = 0; i < count; ++i) {
    if (i) s += ", ";
    s += std::to_string(v[i]);
  }
  return s + "]";
}

std::string quoted_list(const char *b, const char *e, int count) {
  std::string s = "[";
  const char *p = b, *tb, *te;
  for (int i = 0; i < count && next_token(p, e, tb, te); ++i) {
    if (i) s += ", ";
    s += "'";
    s.append(tb, te);
    s += "'";
  }
  return s + "]";
}

struct Chunk {
  const char *b, *e;  // whole lines
  int64_t lines = 0, data = 0;
  int first_fields = -1;  // field count of the chunk's first data line
  int64_t first_line = 0;  // its line index within the chunk (0-based)
  int64_t err_line = -1;   // 0-based within the chunk
  std::string err;
};

std::vector<Chunk> split(const char *text, size_t len, int threads) {
  std::vector<Chunk> ch;
  const size_t per = len / (size_t)threads + 1;
  const char *p = text, *end = text + len;
  while (p < end) {
    const char *q = p + per < end ? p + per : end;
    while (q < end && *(q - 1) != '\n') ++q;  // extend to a line end
    Chunk c;
    c.b = p;
    c.e = q;
    ch.push_back(c);
    p = q;
  }
  return ch;
}

template <typename F>
void for_lines(const Chunk &c, F f) {
  const char *p = c.b;
  int64_t li = 0;
  while (p < c.e) {
    const char *nl = static_cast<const char *>(memchr(p, '\n', (size_t)(c.e - p)));
    const char *le = nl ? nl : c.e;
    if (!f(li, p, le)) return;
    ++li;
    p = nl ? nl + 1 : c.e;
  }
}

void scan_chunk(Chunk &c) {
  for_lines(c, [&](int64_t li, const char *b, const char *e) {
    int fields;
    if (data_line(b, e, &fields)) {
      if (c.first_fields < 0) {
        c.first_fields = fields;
        c.first_line = li;
      }
      ++c.data;
    }
    ++c.lines;
    return true;
  });
}

template <typename F>
void parallel(std::vector<Chunk> &ch, F f) {
  std::vector<std::thread> pool;
  for (size_t i = 1; i < ch.size(); ++i) pool.emplace_back([&, i] { f(ch[i], i); });
  if (!ch.empty()) f(ch[0], 0);
  for (auto &t : pool) t.join();
}

int threads_for(size_t len, int32_t threads) {
  int t = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (t < 1) t = 1;
  const size_t min_chunk = 1 << 20;
  if ((size_t)t > len / min_chunk + 1) t = (int)(len / min_chunk + 1);
  return t;
}

}  // namespace
}  // namespace alto

using namespace alto;

extern "C" {

// Pass 1: number of data lines and the mode count (fields of the first data
// line - 1). *host_err_line = 1-based line of an error, or -1.
int alto_frostt_scan(const char *text, int64_t len, int32_t threads, int64_t *host_entries, int32_t *host_ndim,
                     int64_t *host_err_line) {
  *host_entries = 0;
  *host_ndim = 0;
  *host_err_line = -1;
  std::vector<Chunk> ch = split(text, (size_t)len, threads_for((size_t)len, threads));
  parallel(ch, [](Chunk &c, size_t) { scan_chunk(c); });
  int64_t line0 = 0, entries = 0;
  int ndim = -1;
  for (auto &c : ch) {
    if (ndim < 0 && c.first_fields >= 0) {
      ndim = c.first_fields - 1;
      if (ndim < 1) {
        *host_err_line = line0 + c.first_line + 1;
        set_error("expected at least one index and a value");
        return ALTO_ERR_VALUE;
      }
    }
    line0 += c.lines;
    entries += c.data;
  }
  *host_entries = entries;
  *host_ndim = ndim < 0 ? 0 : ndim;
  return ALTO_OK;
}

// Pass 2: zero-based coords[entries][ndim] (int64) and values[entries]
// (host buffers, typically pinned). First error in file order wins.
int alto_frostt_parse(const char *text, int64_t len, int32_t threads, int32_t ndim, int64_t entries,
                      int64_t *coords, double *values, int64_t *host_err_line) {
  *host_err_line = -1;
  std::vector<Chunk> ch = split(text, (size_t)len, threads_for((size_t)len, threads));
  parallel(ch, [](Chunk &c, size_t) { scan_chunk(c); });
  std::vector<int64_t> out0(ch.size()), line0(ch.size());
  int64_t o = 0, l = 0;
  for (size_t i = 0; i < ch.size(); ++i) {
    out0[i] = o;
    line0[i] = l;
    o += ch[i].data;
    l += ch[i].lines;
  }
  ALTO_REQUIRE(o == entries, ALTO_ERR_VALUE, "entry count changed between scan and parse");
  parallel(ch, [&](Chunk &c, size_t i) {
    int64_t out = out0[i];
    for_lines(c, [&](int64_t li, const char *b, const char *e) {
      int fields;
      if (!data_line(b, e, &fields)) return true;
      auto fail = [&](std::string msg) {
        c.err_line = li;
        c.err = std::move(msg);
        return false;
      };
      if (fields != ndim + 1)
        return fail("expected " + std::to_string(ndim + 1) + " fields, got " + std::to_string(fields));
      const char *p = b, *tb, *te;
      bool nonpos = false;
      long long idx[ALTO_MAX_MODES * 4];
      if (ndim > (int)(sizeof idx / sizeof idx[0])) return fail("too many modes");
      for (int n = 0; n < ndim; ++n) {
        next_token(p, e, tb, te);
        if (!parse_int(tb, te, &idx[n])) return fail("bad index in " + quoted_list(b, e, ndim));
        if (idx[n] <= 0) nonpos = true;
      }
      if (nonpos) return fail("indices are one-based, got " + int_list(idx, ndim));
      for (int n = 0; n < ndim; ++n) coords[out * ndim + n] = idx[n] - 1;
      next_token(p, e, tb, te);
      double v;
      if (!parse_value(tb, te, &v)) return fail("bad value '" + std::string(tb, te) + "'");
      if (!isfinite(v)) return fail("non-finite value '" + std::string(tb, te) + "'");
      values[out] = v;
      ++out;
      return true;
    });
  });
  for (size_t i = 0; i < ch.size(); ++i) {
    if (ch[i].err_line >= 0) {
      *host_err_line = line0[i] + ch[i].err_line + 1;
      set_error("%s", ch[i].err.c_str());
      return ALTO_ERR_VALUE;
    }
  }
  return ALTO_OK;
}

}  // extern "C"
