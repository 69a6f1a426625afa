// Native MatrixMarket entry scanner for the ingestion path (src/io.py:70-163).
//
// The reference splits the whole file into Python strings and parses the
// entry block with np.loadtxt (a slow per-line path exists only to name a
// bad line).  Here one pass over the raw bytes locates the size line and
// parses every entry line into int64 / float64 arrays with their 1-based
// line numbers; the Python wrapper (io.py) keeps the reference's validation
// order and messages, so only the byte crunching moves to C++.
//
// Lines are split on '\n' (a trailing '\r' is whitespace).  A line is
// significant when it is not blank and its first non-blank byte is not '%';
// line 1 (the banner) is never significant.

#include <cerrno>
#include <cstdlib>
#include <cstring>

#include "tb_internal.h"

namespace {

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// [b, e) of the next line starting at *pos; advances *pos past the '\n'.
inline bool next_line(const char *buf, int64_t len, int64_t *pos, int64_t *b, int64_t *e) {
  if (*pos >= len) return false;
  const char *nl = (const char *)memchr(buf + *pos, '\n', (size_t)(len - *pos));
  *b = *pos;
  *e = nl ? nl - buf : len;
  *pos = *e + 1;
  return true;
}

inline bool significant(const char *buf, int64_t b, int64_t e) {
  while (b < e && is_space(buf[b])) ++b;
  return b < e && buf[b] != '%';
}

// Split [b, e) into whitespace-separated fields; returns the count (<= 4 kept).
inline int fields(const char *buf, int64_t b, int64_t e, int64_t fb[4], int64_t fe[4]) {
  int n = 0;
  int64_t p = b;
  while (p < e) {
    while (p < e && is_space(buf[p])) ++p;
    if (p >= e) break;
    const int64_t s = p;
    while (p < e && !is_space(buf[p])) ++p;
    if (n < 4) {
      fb[n] = s;
      fe[n] = p;
    }
    ++n;
  }
  return n;
}

// Copy [b, e) to tmp without Python-style digit-group underscores ("1_000";
// an underscore must sit between two digits).  False if malformed / too long.
inline bool unscore(const char *buf, int64_t b, int64_t e, char *tmp, int cap) {
  int n = 0;
  for (int64_t p = b; p < e; ++p) {
    const char c = buf[p];
    if (c == '_') {
      const bool ok = p > b && p + 1 < e && buf[p - 1] >= '0' && buf[p - 1] <= '9' &&
                      buf[p + 1] >= '0' && buf[p + 1] <= '9';
      if (!ok) return false;
      continue;
    }
    if (n + 1 >= cap) return false;
    tmp[n++] = c;
  }
  tmp[n] = 0;
  return n > 0;
}

// Integer field (Python int(): optional sign, digits, digit-group
// underscores); "1.0" or "x" fail.
inline bool parse_int(const char *buf, int64_t b, int64_t e, int64_t *out) {
  char tmp[64];
  if (!unscore(buf, b, e, tmp, (int)sizeof(tmp))) return false;
  const char *p = tmp;
  bool neg = false;
  if (*p == '+' || *p == '-') neg = *p++ == '-';
  if (!*p) return false;
  int64_t v = 0;
  for (; *p; ++p) {
    if (*p < '0' || *p > '9') return false;
    v = v * 10 + (*p - '0');
  }
  *out = neg ? -v : v;
  return true;
}

// Real field (Python float(): decimal / exponent / inf / nan, digit-group
// underscores; no hexadecimal, which strtod alone would accept).
inline bool parse_real(const char *buf, int64_t b, int64_t e, double *out) {
  char tmp[128];
  if (!unscore(buf, b, e, tmp, (int)sizeof(tmp))) return false;
  for (const char *q = tmp; *q; ++q)
    if (*q == 'x' || *q == 'X' || *q == '(') return false;
  char *end = nullptr;
  errno = 0;
  const double v = strtod(tmp, &end);
  if (*end != 0 || end == tmp) return false;
  *out = v;
  return true;
}

}  // namespace

// Locate the size line: its 1-based number and byte range (size_line = 0 if
// the file has no significant line after the banner).  *lines = total lines.
extern "C" int tb_mm_locate(const char *buf, int64_t len, int64_t *size_line, int64_t *size_b,
                            int64_t *size_e, int64_t *body_pos, int64_t *lines) {
  *size_line = 0;
  *size_b = *size_e = *body_pos = 0;
  int64_t pos = 0, b, e, no = 0;
  while (next_line(buf, len, &pos, &b, &e)) {
    ++no;
    if (no > 1 && !*size_line && significant(buf, b, e)) {
      *size_line = no;
      *size_b = b;
      *size_e = e;
      *body_pos = pos;
    }
  }
  *lines = no;
  return TB_OK;
}

// Parse the entry lines after the size line (starting at byte body_pos,
// whose line number is first_line).  Up to `cap` entries are stored; *found
// counts all significant lines.  *kth_line = line number of significant
// line number `cap` (0-based; the first surplus line) or 0.
// Field errors are reported for the first bad line among the first `cap`:
// *err_kind 1 = not three fields, 2 = bad index, 3 = non-real value, with
// its line number and the byte range of the failing field / line.
extern "C" int tb_mm_entries(const char *buf, int64_t len, int64_t body_pos, int64_t first_line,
                             int64_t cap, int64_t *rows, int64_t *cols, double *vals,
                             int64_t *linenos, int64_t *found, int64_t *kth_line,
                             int32_t *err_kind, int64_t *err_line, int64_t *err_b,
                             int64_t *err_e) {
  *found = 0;
  *kth_line = 0;
  *err_kind = 0;
  *err_line = 0;
  *err_b = *err_e = 0;
  int64_t pos = body_pos, b, e, no = first_line - 1;
  int64_t soft_line = 0, soft_b = 0, soft_e = 0;
  while (next_line(buf, len, &pos, &b, &e)) {
    ++no;
    if (!significant(buf, b, e)) continue;
    const int64_t k = (*found)++;
    if (k == cap) *kth_line = no;
    if (k >= cap || *err_kind) continue;
    int64_t fb[4], fe[4];
    const int nf = fields(buf, b, e, fb, fe);
    int kind = 0;
    int64_t eb = b, ee = e;
    bool soft = false;
    auto index = [&](int f, int64_t *out) {
      if (parse_int(buf, fb[f], fe[f], out)) return true;
      // "2.0": the reference's np.loadtxt fast path accepts integral reals
      // as indices -- but only when every entry line parses that way
      double r;
      if (parse_real(buf, fb[f], fe[f], &r) && r == (double)(int64_t)r) {
        *out = (int64_t)r;
        soft = true;
        return true;
      }
      return false;
    };
    if (nf != 3) {
      kind = 1;
    } else if (!index(0, &rows[k]) || !index(1, &cols[k])) {
      kind = 2;
    } else if (!parse_real(buf, fb[2], fe[2], &vals[k])) {
      kind = 3;
      eb = fb[2];
      ee = fe[2];
    }
    if (soft && !kind && !soft_line) {
      soft_line = no;
      soft_b = b;
      soft_e = e;
    }
    if (kind) {
      *err_kind = kind;
      *err_line = no;
      if (kind != 3) {  // the stripped line
        while (eb < ee && is_space(buf[eb])) ++eb;
        while (ee > eb && is_space(buf[ee - 1])) --ee;
      }
      *err_b = eb;
      *err_e = ee;
      continue;
    }
    linenos[k] = no;
  }
  // the reference's slow path (taken once any line fails) rejects integral
  // reals as indices: report whichever comes first
  if (*err_kind && soft_line && soft_line < *err_line) {
    *err_kind = 2;
    *err_line = soft_line;
    while (soft_b < soft_e && is_space(buf[soft_b])) ++soft_b;
    while (soft_e > soft_b && is_space(buf[soft_e - 1])) --soft_e;
    *err_b = soft_b;
    *err_e = soft_e;
  }
  return TB_OK;
}
