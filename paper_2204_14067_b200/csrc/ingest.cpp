// Native ratings-text ingest: a multi-threaded
// parser for the whitespace "user item rating [timestamp]" format that
// mfg/data.py:164-200 (_parse_stream) reads line by line in Python.
//
// The parser accepts exactly the lines whose Python parse is unambiguous:
// ASCII, fields separated by ASCII whitespace, 3 or 4 fields, ids made of
// decimal digits and > 0, the rating a plain decimal float. Values are
// identical to Python's int()/float() (std::from_chars is correctly rounded,
// as float() is). Any other line -- a malformed one, a non-positive id, a
// sign, underscores, "inf", non-ASCII bytes -- stops the fast path: the call
// returns MFG_ERR_ARG with *first_odd_line set, and the caller re-parses the
// input with the reference's own logic, which either accepts the line or
// raises the reference's exact error. Empty (whitespace-only) lines are
// skipped and counted, as in the reference.

#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/mfg_b200.h"

namespace {

// Python str.split()/strip() whitespace within ASCII: \t \n \v \f \r, space,
// and \x1c-\x1f.
inline bool is_ws(unsigned char c) {
  return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f);
}

struct Chunk {
  const char* b;
  const char* e;
  int64_t first_line;  // 1-based number of the chunk's first line
  std::vector<int64_t> u, i;
  std::vector<double> r;
  int64_t odd = 0;     // first line the fast path cannot take (0 = none)
};

bool parse_id(const char* s, const char* e, int64_t* out) {
  if (s == e || e - s > 18) return false;
  int64_t v = 0;
  for (const char* p = s; p < e; ++p) {
    if (*p < '0' || *p > '9') return false;
    v = v * 10 + (*p - '0');
  }
  if (v <= 0) return false;
  *out = v;
  return true;
}

bool parse_rating(const char* s, const char* e, double* out) {
  // plain decimal: [+-]? digits [. digits] [(e|E) [+-]? digits], at least one digit
  const char* p = s;
  if (p < e && (*p == '+' || *p == '-')) ++p;
  const char* d0 = p;
  while (p < e && *p >= '0' && *p <= '9') ++p;
  bool digits = p > d0;
  if (p < e && *p == '.') {
    ++p;
    const char* f0 = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    digits = digits || p > f0;
  }
  if (!digits) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    ++p;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    const char* x0 = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    if (p == x0) return false;
  }
  if (p != e) return false;
  const char* q = s + (*s == '+' ? 1 : 0);  // from_chars rejects a leading '+'
  auto res = std::from_chars(q, e, *out, std::chars_format::general);
  return res.ec == std::errc() && res.ptr == e;
}

void parse_chunk(Chunk& c) {
  const char* p = c.b;
  int64_t line = c.first_line;
  while (p < c.e) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', c.e - p));
    const char* le = nl ? nl : c.e;
    const char* f[5][2];
    int nf = 0;
    const char* q = p;
    bool ok = true;
    while (q < le) {
      const unsigned char ch = static_cast<unsigned char>(*q);
      if (ch >= 0x80 || (ch < 0x20 && !is_ws(ch)) || ch == 0x7f) { ok = false; break; }
      if (is_ws(ch)) { ++q; continue; }
      const char* s = q;
      while (q < le && !is_ws(static_cast<unsigned char>(*q))) {
        const unsigned char c2 = static_cast<unsigned char>(*q);
        if (c2 >= 0x80 || c2 < 0x20 || c2 == 0x7f) { ok = false; break; }
        ++q;
      }
      if (!ok) break;
      if (nf < 5) { f[nf][0] = s; f[nf][1] = q; }
      ++nf;
    }
    if (ok && nf != 0) {
      int64_t u = 0, i = 0;
      double r = 0.0;
      ok = (nf == 3 || nf == 4) && parse_id(f[0][0], f[0][1], &u) &&
           parse_id(f[1][0], f[1][1], &i) && parse_rating(f[2][0], f[2][1], &r);
      if (ok) {
        c.u.push_back(u);
        c.i.push_back(i);
        c.r.push_back(r);
      }
    }
    if (!ok) { c.odd = line; return; }
    ++line;
    p = nl ? nl + 1 : c.e;
  }
}

}  // namespace

extern "C" int64_t mfg_count_lines(const char* buf, size_t len) {
  if (!buf || len == 0) return 0;
  int64_t n = 0;
  const char* p = buf;
  const char* e = buf + len;
  while ((p = static_cast<const char*>(memchr(p, '\n', e - p)))) { ++n; ++p; }
  return n + (buf[len - 1] != '\n' ? 1 : 0);
}

extern "C" int mfg_parse_ratings(const char* buf, size_t len, int nthreads, int64_t* users,
                                 int64_t* items, double* ratings, size_t cap, size_t* count,
                                 int64_t* first_odd_line) {
  if (!count || !first_odd_line || (len && !buf)) return MFG_ERR_ARG;
  *count = 0;
  *first_odd_line = 0;
  if (len == 0) return MFG_OK;
  int nt = nthreads > 0 ? nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::min<size_t>((size_t)nt, std::max<size_t>(1, len / (1 << 20)));  // >= 1 MiB per thread
  // chunk boundaries just after a '\n'
  std::vector<const char*> cut(nt + 1);
  cut[0] = buf;
  cut[nt] = buf + len;
  for (int t = 1; t < nt; ++t) {
    const char* g = buf + len * t / nt;
    if (g < cut[t - 1]) g = cut[t - 1];
    const char* nl = static_cast<const char*>(memchr(g, '\n', buf + len - g));
    cut[t] = nl ? nl + 1 : buf + len;
  }
  std::vector<Chunk> ch(nt);
  std::vector<int64_t> lines(nt, 0);
  auto count_nl = [](const char* b, const char* e) {
    int64_t n = 0;
    while (b < e && (b = static_cast<const char*>(memchr(b, '\n', e - b)))) { ++n; ++b; }
    return n;
  };
  {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] { lines[t] = count_nl(cut[t], cut[t + 1]); });
    for (auto& x : th) x.join();
  }
  int64_t first = 1;
  for (int t = 0; t < nt; ++t) {
    ch[t].b = cut[t];
    ch[t].e = cut[t + 1];
    ch[t].first_line = first;
    first += lines[t];
  }
  {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back([&, t] { parse_chunk(ch[t]); });
    for (auto& x : th) x.join();
  }
  for (int t = 0; t < nt; ++t)
    if (ch[t].odd) { *first_odd_line = ch[t].odd; return MFG_ERR_ARG; }
  size_t total = 0;
  for (auto& c : ch) total += c.u.size();
  if (total > cap) return MFG_ERR_CAPACITY;
  size_t off = 0;
  for (auto& c : ch) {
    std::copy(c.u.begin(), c.u.end(), users + off);
    std::copy(c.i.begin(), c.i.end(), items + off);
    std::copy(c.r.begin(), c.r.end(), ratings + off);
    off += c.u.size();
  }
  *count = total;
  return MFG_OK;
}
