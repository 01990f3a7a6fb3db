// Dataset text loaders (io.py:16-77): libsvm and CSV -> dense row-major f32/f64,
// host side of the GPU path (the parsed matrix is what run_lloyd copies to HBM).
//
// Semantics follow the reference loaders line for line, so results and the
// FIRST error reported are the same:
//   * text mode with universal newlines: "\n", "\r\n" and a lone "\r" end a
//     line; physical line numbers start at 1 and count blank lines;
//   * a line is blank when str.strip() leaves nothing (ASCII whitespace
//     " \t\n\r\v\f" and \x1c-\x1f, which str.isspace() also accepts);
//   * numbers are parsed with Python's float() grammar (optional surrounding
//     whitespace, sign, digits with single '_' separators, '.', exponent,
//     inf/infinity/nan in any case) and rounded correctly to double
//     (std::from_chars), then to f32 when the output is f32 — exactly what
//     float(text) followed by a store into an f32 numpy array does;
//   * libsvm: first n non-blank lines; token 0 = class label (must parse,
//     discarded), then idx:val pairs with 1 <= int(idx) <= d, later duplicates
//     win; lines after the n-th are not read (io.py:16-46);
//   * CSV: every non-blank line is parsed (so an error past row n is still
//     reported before the row-count check); a first line with any non-numeric
//     cell is a header and skipped (io.py:49-77).
// Non-ASCII input is treated byte-wise (Unicode digits/spaces that Python's
// float()/int()/split() would accept are rejected here).
//
// Lines are located in one sequential pass, then parsed by a pool of threads;
// each thread records the first error of its range and the error with the
// smallest line number wins, which is the one the sequential reference hits.
// Errors are returned as (kind, line number, offending text) and formatted by
// the Python layer with the reference's exact messages.
#include <algorithm>
#include <atomic>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <sys/stat.h>
#include <string>
#include <thread>
#include <vector>

namespace {

enum ErrKind : int64_t {
  kOk = 0,
  kLibsvmLabel = 1,      // malformed label {tok!r}
  kLibsvmToken = 2,      // malformed feature token {tok!r}
  kLibsvmIndex = 3,      // feature index {int(tok)} out of range [1, d]   (tok = idx text)
  kLibsvmTooFew = 4,     // expected {n} data lines, found {count}
  kCsvEmpty = 5,         // file is empty
  kCsvCell = 6,          // non-numeric cell in row {text!r}
  kCsvColumns = 7,       // expected {d} columns, found {count}
  kCsvRows = 8,          // expected {n} data rows, found {count}
};

constexpr int PCB_EINVAL = -1;
constexpr int PCB_EPARSE = -4;

inline bool is_ws(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f);
}

struct Span {
  const char* b;
  const char* e;
  size_t size() const { return (size_t)(e - b); }
};

inline Span strip(Span s) {
  while (s.b < s.e && is_ws((unsigned char)*s.b)) ++s.b;
  while (s.e > s.b && is_ws((unsigned char)s.e[-1])) --s.e;
  return s;
}

inline bool ieq(const char* a, size_t n, const char* lit) {
  if (strlen(lit) != n) return false;
  for (size_t i = 0; i < n; ++i)
    if ((char)tolower((unsigned char)a[i]) != lit[i]) return false;
  return true;
}

// digitpart := digit (['_'] digit)*  ; appends the digits to buf
inline bool digitpart(const char*& p, const char* e, std::string& buf) {
  if (p >= e || !isdigit((unsigned char)*p)) return false;
  buf.push_back(*p++);
  while (p < e) {
    if (isdigit((unsigned char)*p)) {
      buf.push_back(*p++);
    } else if (*p == '_' && p + 1 < e && isdigit((unsigned char)p[1])) {
      ++p;
    } else {
      break;
    }
  }
  return true;
}

// Python float(text) -> double; false if float() would raise ValueError.
bool py_float(Span s, double& out, std::string& buf) {
  s = strip(s);
  const char* p = s.b;
  const char* e = s.e;
  if (p >= e) return false;
  bool neg = false;
  if (*p == '+' || *p == '-') neg = (*p++ == '-');
  const size_t rest = (size_t)(e - p);
  if (ieq(p, rest, "inf") || ieq(p, rest, "infinity")) {
    out = neg ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(p, rest, "nan")) {
    out = neg ? -NAN : NAN;
    return true;
  }
  buf.clear();
  bool intpart = digitpart(p, e, buf);
  bool frac = false;
  if (p < e && *p == '.') {
    buf.push_back('.');
    ++p;
    frac = digitpart(p, e, buf);
  }
  if (!intpart && !frac) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    buf.push_back('e');
    ++p;
    if (p < e && (*p == '+' || *p == '-')) buf.push_back(*p++);
    if (!digitpart(p, e, buf)) return false;
  }
  if (p != e) return false;
  double v = 0.0;
  auto r = std::from_chars(buf.data(), buf.data() + buf.size(), v, std::chars_format::general);
  if (r.ec == std::errc::result_out_of_range) {
    // Python rounds overflow to inf and underflow to (signed) zero without error
    // (strtod semantics); from_chars reports the range error instead
    v = strtod(std::string(buf).c_str(), nullptr);
  } else if (r.ec != std::errc() || r.ptr != buf.data() + buf.size()) {
    return false;
  }
  out = neg ? -v : v;
  return true;
}

// Python int(text) for a base-10 string -> int64 (saturating; the caller only
// range-checks it).  false if int() would raise ValueError.
bool py_int(Span s, int64_t& out, std::string& buf) {
  s = strip(s);
  const char* p = s.b;
  const char* e = s.e;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = (*p++ == '-');
  buf.clear();
  if (!digitpart(p, e, buf) || p != e) return false;
  int64_t v = 0;
  for (char c : buf) {
    if (v > (INT64_MAX - 9) / 10) {
      v = INT64_MAX;
      break;
    }
    v = v * 10 + (c - '0');
  }
  out = neg ? -v : v;
  return true;
}

struct FileText {
  std::vector<char> data;
  std::vector<Span> lines;       // every physical line (terminator excluded)
};

int read_lines(const char* path, FileText& ft) {
  FILE* f = fopen(path, "rb");
  if (!f) return errno ? errno : EIO;
  struct stat stt;
  if (fstat(fileno(f), &stt) == 0 && S_ISDIR(stt.st_mode)) {
    fclose(f);
    return EISDIR;
  }
  if (fseek(f, 0, SEEK_END) != 0) { int e = errno; fclose(f); return e ? e : EIO; }
  long sz = ftell(f);
  if (sz < 0) { int e = errno; fclose(f); return e ? e : EIO; }
  rewind(f);
  ft.data.resize((size_t)sz);
  if (sz > 0 && fread(ft.data.data(), 1, (size_t)sz, f) != (size_t)sz) { fclose(f); return EIO; }
  fclose(f);
  const char* p = ft.data.data();
  const char* e = p + ft.data.size();
  const char* start = p;
  while (p < e) {
    const char c = *p;
    if (c == '\n' || c == '\r') {
      ft.lines.push_back(Span{start, p});
      if (c == '\r' && p + 1 < e && p[1] == '\n') ++p;
      start = ++p;
    } else {
      ++p;
    }
  }
  if (start < e) ft.lines.push_back(Span{start, e});
  return 0;
}

struct Err {
  int64_t kind = kOk;
  int64_t lineno = INT64_MAX;
  int64_t count = 0;
  std::string text;
};

inline void note(Err& err, int64_t kind, int64_t lineno, Span t) {
  if (lineno < err.lineno) {
    err.kind = kind;
    err.lineno = lineno;
    err.text.assign(t.b, t.e);
  }
}

int pick_threads(int requested, size_t items) {
  int t = requested > 0 ? requested : (int)std::thread::hardware_concurrency();
  t = std::max(1, std::min(t, 64));
  return (int)std::min<size_t>((size_t)t, std::max<size_t>(1, items / 1024));
}

template <typename F>
void parallel_ranges(size_t items, int threads, F&& fn) {
  if (threads <= 1) {
    fn(0, 0, items);
    return;
  }
  std::vector<std::thread> pool;
  const size_t per = (items + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const size_t lo = std::min(items, (size_t)t * per), hi = std::min(items, lo + per);
    pool.emplace_back([&fn, t, lo, hi] { fn(t, lo, hi); });
  }
  for (auto& th : pool) th.join();
}

void report(const Err& err, int64_t* info, char* text, int64_t text_len) {
  info[0] = err.kind;
  info[1] = err.lineno == INT64_MAX ? 0 : err.lineno;
  info[2] = err.count;
  if (text && text_len > 0) {
    const size_t m = std::min<size_t>(err.text.size(), (size_t)text_len - 1);
    memcpy(text, err.text.data(), m);
    text[m] = '\0';
    info[3] = (int64_t)err.text.size();
  }
}

template <typename T>
int load_libsvm_t(const char* path, int64_t n, int d, T* out, int64_t* info, char* text, int64_t text_len,
                  int nthreads) {
  FileText ft;
  if (int e = read_lines(path, ft)) return e;
  // the first n non-blank lines (line numbers are physical)
  std::vector<std::pair<Span, int64_t>> rows;
  rows.reserve((size_t)n);
  for (size_t i = 0; i < ft.lines.size() && (int64_t)rows.size() < n; ++i) {
    Span s = strip(ft.lines[i]);
    if (s.size()) rows.push_back({s, (int64_t)i + 1});
  }
  const int T_ = pick_threads(nthreads, rows.size());
  std::vector<Err> errs((size_t)T_);
  parallel_ranges(rows.size(), T_, [&](int t, size_t lo, size_t hi) {
    std::string buf;
    Err& err = errs[(size_t)t];
    for (size_t r = lo; r < hi && err.kind == kOk; ++r) {
      const Span line = rows[r].first;
      const int64_t lineno = rows[r].second;
      const char* p = line.b;
      auto next_token = [&](Span& tok) {
        while (p < line.e && is_ws((unsigned char)*p)) ++p;
        if (p >= line.e) return false;
        tok.b = p;
        while (p < line.e && !is_ws((unsigned char)*p)) ++p;
        tok.e = p;
        return true;
      };
      Span tok;
      next_token(tok);
      double v;
      if (!py_float(tok, v, buf)) { note(err, kLibsvmLabel, lineno, tok); break; }
      T* row = out + (int64_t)r * d;
      while (next_token(tok)) {
        const char* colon = (const char*)memchr(tok.b, ':', tok.size());
        int64_t idx;
        if (!colon || !py_int(Span{tok.b, colon}, idx, buf) || !py_float(Span{colon + 1, tok.e}, v, buf)) {
          note(err, kLibsvmToken, lineno, tok);
          break;
        }
        if (idx < 1 || idx > d) {
          note(err, kLibsvmIndex, lineno, Span{tok.b, colon});
          break;
        }
        row[idx - 1] = (T)v;
      }
    }
  });
  Err first;
  for (auto& e : errs)
    if (e.kind != kOk && e.lineno < first.lineno) first = e;
  if (first.kind == kOk && (int64_t)rows.size() < n) {
    first.kind = kLibsvmTooFew;
    first.count = (int64_t)rows.size();
  }
  report(first, info, text, text_len);
  return first.kind == kOk ? 0 : PCB_EPARSE;
}

template <typename T>
int load_csv_t(const char* path, int64_t n, int d, T* out, int64_t* info, char* text, int64_t text_len,
               int nthreads) {
  FileText ft;
  if (int e = read_lines(path, ft)) return e;
  std::vector<std::pair<Span, int64_t>> rows;
  for (size_t i = 0; i < ft.lines.size(); ++i) {
    Span s = strip(ft.lines[i]);
    if (s.size()) rows.push_back({s, (int64_t)i + 1});
  }
  Err first;
  if (rows.empty()) {
    first.kind = kCsvEmpty;
    report(first, info, text, text_len);
    return PCB_EPARSE;
  }
  // header: any cell of the first line that float() rejects
  size_t start = 0;
  {
    std::string buf;
    const Span h = rows[0].first;
    const char* c = h.b;
    while (true) {
      const char* comma = (const char*)memchr(c, ',', (size_t)(h.e - c));
      const char* ce = comma ? comma : h.e;
      double v;
      if (!py_float(Span{c, ce}, v, buf)) { start = 1; break; }
      if (!comma) break;
      c = comma + 1;
    }
  }
  const size_t nrows = rows.size() - start;
  const int T_ = pick_threads(nthreads, nrows);
  std::vector<Err> errs((size_t)T_);
  parallel_ranges(nrows, T_, [&](int t, size_t lo, size_t hi) {
    std::string buf;
    Err& err = errs[(size_t)t];
    for (size_t r = lo; r < hi && err.kind == kOk; ++r) {
      const Span line = rows[start + r].first;
      const int64_t lineno = rows[start + r].second;
      const char* c = line.b;
      int64_t col = 0;
      const bool store = (int64_t)r < n;
      while (true) {
        const char* comma = (const char*)memchr(c, ',', (size_t)(line.e - c));
        const char* ce = comma ? comma : line.e;
        double v;
        if (!py_float(Span{c, ce}, v, buf)) { note(err, kCsvCell, lineno, line); break; }
        if (store && col < d) out[(int64_t)r * d + col] = (T)v;
        ++col;
        if (!comma) break;
        c = comma + 1;
      }
      if (err.kind == kOk && col != d) {
        note(err, kCsvColumns, lineno, Span{line.b, line.b});
        err.count = col;
      }
    }
  });
  for (auto& e : errs)
    if (e.kind != kOk && e.lineno < first.lineno) first = e;
  if (first.kind == kOk && (int64_t)nrows != n) {
    first.kind = kCsvRows;
    first.count = (int64_t)nrows;
  }
  report(first, info, text, text_len);
  return first.kind == kOk ? 0 : PCB_EPARSE;
}

}  // namespace

extern "C" {

// Returns 0, a positive errno (file could not be read), PCB_EINVAL, or
// PCB_EPARSE with info = {kind, line number, count, text length} and the
// offending text in `text` (NUL-terminated, truncated to text_len - 1).
int pcb_load_libsvm(const char* path, int64_t n, int d, int is_f64, void* out_host, int64_t* info, char* text,
                    int64_t text_len, int nthreads) {
  if (!path || n < 0 || d < 0 || (n > 0 && d > 0 && !out_host) || !info) return PCB_EINVAL;
  info[0] = info[1] = info[2] = info[3] = 0;
  return is_f64 ? load_libsvm_t(path, n, d, (double*)out_host, info, text, text_len, nthreads)
                : load_libsvm_t(path, n, d, (float*)out_host, info, text, text_len, nthreads);
}

int pcb_load_csv(const char* path, int64_t n, int d, int is_f64, void* out_host, int64_t* info, char* text,
                 int64_t text_len, int nthreads) {
  if (!path || n < 0 || d < 0 || (n > 0 && d > 0 && !out_host) || !info) return PCB_EINVAL;
  info[0] = info[1] = info[2] = info[3] = 0;
  return is_f64 ? load_csv_t(path, n, d, (double*)out_host, info, text, text_len, nthreads)
                : load_csv_t(path, n, d, (float*)out_host, info, text, text_len, nthreads);
}

}  // extern "C"
