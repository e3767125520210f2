// Plain-text problem file ("BAL" layout) reader / writer, host side, multi-threaded.
//
// Reference: pkg/src/bamg/balio.py:25-97 (write_bal / read_bal / BalFormatError).
// Layout: header "n_cameras n_points n_observations"; one line "camera point x y"
// per observation; then 9 scalar lines per camera and 3 per point. Blank lines are
// skipped anywhere. Errors carry the 1-based line number and the reference's
// message text; the first error in file order wins, as in the sequential reader.
//
// The file is mapped once; pass 1 counts lines and non-blank lines per chunk (chunk
// boundaries sit after a '\n'); pass 2 knows from those counts which record every
// non-blank line is, so chunks parse independently. Numbers use std::from_chars
// (correctly rounded, so a %.17g write / read round trip is bit-exact).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bamg_b200.h"

namespace {

// Python str.splitlines() boundaries (ASCII subset); "\r\n" is one boundary
inline bool is_break(char c) { return c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1e); }
// str.split() / str.strip() whitespace inside a line (ASCII subset)
inline bool is_space(char c) { return c == ' ' || c == '\t' || c == 0x1f; }

struct Line {
  const char* b;
  const char* e;
};

// next line starting at p (< end); returns the line and advances p past its break
inline Line next_raw_line(const char*& p, const char* end) {
  const char* s = p;
  while (p < end && !is_break(*p)) ++p;
  Line l{s, p};
  if (p < end) {
    if (*p == '\r' && p + 1 < end && p[1] == '\n') ++p;
    ++p;
  }
  return l;
}

inline Line strip(Line l) {
  while (l.b < l.e && is_space(*l.b)) ++l.b;
  while (l.e > l.b && is_space(l.e[-1])) --l.e;
  return l;
}

inline int split(Line l, Line* parts, int maxp) {
  int n = 0;
  const char* p = l.b;
  while (p < l.e) {
    while (p < l.e && is_space(*p)) ++p;
    if (p >= l.e) break;
    const char* s = p;
    while (p < l.e && !is_space(*p)) ++p;
    if (n < maxp) parts[n] = Line{s, p};
    ++n;
  }
  return n;
}

// Python's underscore rule: single '_' only between two digits
bool strip_underscores(Line t, std::string& out) {
  out.clear();
  for (const char* p = t.b; p < t.e; ++p) {
    if (*p == '_') {
      if (p == t.b || p + 1 >= t.e || !isdigit((unsigned char)p[-1]) || !isdigit((unsigned char)p[1])) return false;
      continue;
    }
    out.push_back(*p);
  }
  return true;
}

// int(token): [+-]digits (underscores between digits). Sets `big` on int64 overflow.
bool parse_int(Line t, long long& v, bool& big, std::string& norm) {
  std::string s;
  if (!strip_underscores(t, s) || s.empty()) return false;
  size_t i = 0;
  bool neg = false;
  if (s[0] == '+' || s[0] == '-') {
    neg = s[0] == '-';
    i = 1;
  }
  if (i >= s.size()) return false;
  for (size_t k = i; k < s.size(); ++k)
    if (!isdigit((unsigned char)s[k])) return false;
  size_t nz = i;
  while (nz + 1 < s.size() && s[nz] == '0') ++nz;
  norm = std::string(neg && !(s.size() - nz == 1 && s[nz] == '0') ? "-" : "") + s.substr(nz);
  big = false;
  unsigned long long acc = 0;
  for (size_t k = i; k < s.size(); ++k) {
    unsigned d = (unsigned)(s[k] - '0');
    if (acc > (9223372036854775807ull - d) / 10) {
      big = true;
      break;
    }
    acc = acc * 10 + d;
  }
  v = big ? 0 : (neg ? -(long long)acc : (long long)acc);
  return true;
}

// float(token): optional sign, decimal / exponent / inf / infinity / nan
bool parse_float(Line t, double& v) {
  std::string s;
  if (!strip_underscores(t, s) || s.empty()) return false;
  const char* b = s.data();
  const char* e = b + s.size();
  bool neg = false;
  if (*b == '+' || *b == '-') {
    neg = *b == '-';
    ++b;
  }
  if (b >= e || *b == '+' || *b == '-') return false;
  for (const char* p = b; p < e; ++p)
    if (*p == '(') return false;  // from_chars accepts nan(...), float() does not
  auto r = std::from_chars(b, e, v, std::chars_format::general);
  if (r.ec == std::errc::result_out_of_range) {
    // float() rounds to 0 / inf rather than failing
    v = strtod(std::string(b, e).c_str(), nullptr);
  } else if (r.ec != std::errc() || r.ptr != e) {
    return false;
  }
  if (neg) v = -v;
  return true;
}

std::string py_repr(Line l) {
  std::string s(l.b, l.e);
  char q = (s.find('\'') != std::string::npos && s.find('"') == std::string::npos) ? '"' : '\'';
  std::string out(1, q);
  for (unsigned char c : s) {
    if (c == '\\') out += "\\\\";
    else if (c == (unsigned char)q) out += std::string("\\") + (char)q;
    else if (c == '\t') out += "\\t";
    else if (c == '\n') out += "\\n";
    else if (c == '\r') out += "\\r";
    else if (c < 0x20 || c == 0x7f) {
      char buf[8];
      snprintf(buf, sizeof buf, "\\x%02x", c);
      out += buf;
    } else out += (char)c;
  }
  out += q;
  return out;
}

struct Mapped {
  const char* p = nullptr;
  size_t n = 0;
  int fd = -1;
  ~Mapped() {
    if (p && n) munmap((void*)p, n);
    if (fd >= 0) close(fd);
  }
};

int map_file(const char* path, Mapped& m) {
  m.fd = open(path, O_RDONLY);
  if (m.fd < 0) return -errno;
  struct stat st;
  if (fstat(m.fd, &st) != 0) return -errno;
  m.n = (size_t)st.st_size;
  if (m.n == 0) return 0;
  void* a = mmap(nullptr, m.n, PROT_READ, MAP_PRIVATE, m.fd, 0);
  if (a == MAP_FAILED) return -errno;
  madvise(a, m.n, MADV_SEQUENTIAL);
  m.p = (const char*)a;
  return 0;
}

void set_err(long long line, const std::string& msg, long long* err_line, char* err_msg, size_t err_len) {
  if (err_line) *err_line = line;
  if (err_msg && err_len) {
    size_t k = std::min(err_len - 1, msg.size());
    memcpy(err_msg, msg.data(), k);
    err_msg[k] = 0;
  }
}

int threads_for(int requested, size_t bytes) {
  int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  int t = requested > 0 ? requested : hw;
  size_t cap = std::max<size_t>(1, bytes / (1 << 20));  // >= 1 MB per thread
  return (int)std::max<size_t>(1, std::min<size_t>((size_t)t, cap));
}

// header: first non-blank line -> counts (balio.py:56-66)
int parse_header(const char* p, const char* end, long long counts[3], long long* hdr_line, long long* err_line,
                 char* err_msg, size_t err_len) {
  long long lineno = 0;
  while (p < end) {
    Line l = strip(next_raw_line(p, end));
    ++lineno;
    if (l.b == l.e) continue;
    *hdr_line = lineno;
    Line parts[4];
    int n = split(l, parts, 4);
    if (n != 3) {
      set_err(lineno, "header needs 3 counts, got " + std::to_string(n), err_line, err_msg, err_len);
      return BAMG_ERR_FORMAT;
    }
    for (int k = 0; k < 3; ++k) {
      long long v;
      bool big;
      std::string norm;
      if (!parse_int(parts[k], v, big, norm)) {
        set_err(lineno, "malformed header count in " + py_repr(l), err_line, err_msg, err_len);
        return BAMG_ERR_FORMAT;
      }
      if (big) {
        set_err(lineno, "header count " + norm + " is too large", err_line, err_msg, err_len);
        return BAMG_ERR_FORMAT;
      }
      counts[k] = v;
    }
    if (counts[0] < 0 || counts[1] < 0 || counts[2] < 0) {
      set_err(lineno, "counts must be nonnegative", err_line, err_msg, err_len);
      return BAMG_ERR_FORMAT;
    }
    return 0;
  }
  set_err(lineno + 1, "file ends before header", err_line, err_msg, err_len);
  return BAMG_ERR_FORMAT;
}

struct Chunk {
  const char* b;
  const char* e;
  long long lines = 0, nonblank = 0;      // pass 1
  long long line0 = 0, nb0 = 0;           // prefix (lines / non-blank before the chunk)
  long long err_line = -1;                // pass 2: first error in this chunk
  std::string err;
  long long last_line = -1;               // line holding the last expected record
  bool trailing = false;
};

}  // namespace

extern "C" int bamg_bal_read_header(const char* path, int64_t* counts, int64_t* err_line, char* err_msg,
                                    size_t err_len) {
  Mapped m;
  int rc = map_file(path, m);
  if (rc) {
    set_err(0, std::string("cannot read ") + path + ": " + strerror(-rc), (long long*)err_line, err_msg, err_len);
    return BAMG_ERR_CUDA;
  }
  long long c[3], hl;
  rc = parse_header(m.p, m.p + m.n, c, &hl, (long long*)err_line, err_msg, err_len);
  if (rc) return rc;
  for (int k = 0; k < 3; ++k) counts[k] = c[k];
  return 0;
}

extern "C" int bamg_bal_read(const char* path, int64_t n_cam, int64_t n_pt, int64_t n_obs, int64_t* cam_index,
                             int64_t* pt_index, double* pixels, double* cams, double* pts, int32_t n_threads,
                             int64_t* err_line, char* err_msg, size_t err_len) {
  Mapped m;
  int rc = map_file(path, m);
  if (rc) {
    set_err(0, std::string("cannot read ") + path + ": " + strerror(-rc), (long long*)err_line, err_msg, err_len);
    return BAMG_ERR_CUDA;
  }
  const char* p0 = m.p;
  const char* end = m.p + m.n;
  long long hc[3], hdr_line = 0;
  rc = parse_header(p0, end, hc, &hdr_line, (long long*)err_line, err_msg, err_len);
  if (rc) return rc;
  if (hc[0] != n_cam || hc[1] != n_pt || hc[2] != n_obs) {
    set_err(hdr_line, "header counts differ from the caller's", (long long*)err_line, err_msg, err_len);
    return BAMG_ERR_FORMAT;
  }
  // record k (k = non-blank index): 0 header, 1..n_obs observations, then 9 n_cam
  // camera scalars, then 3 n_pt point scalars
  const long long n_rec = 1 + n_obs + 9 * n_cam + 3 * n_pt;
  int T = threads_for(n_threads, m.n);
  std::vector<Chunk> ch(T);
  for (int t = 0; t < T; ++t) {
    const char* b = (t == 0) ? p0 : p0 + m.n * t / T;
    if (t > 0) {
      while (b < end && b[-1] != '\n') ++b;
    }
    ch[t].b = b;
  }
  for (int t = 0; t < T; ++t) ch[t].e = (t + 1 < T) ? std::max(ch[t].b, ch[t + 1].b) : end;
  auto pass1 = [&](int t) {
    Chunk& c = ch[t];
    const char* p = c.b;
    while (p < c.e) {
      Line l = strip(next_raw_line(p, c.e));
      ++c.lines;
      if (l.b != l.e) ++c.nonblank;
    }
  };
  auto run = [&](auto fn) {
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(fn, t);
    fn(0);
    for (auto& x : th) x.join();
  };
  run(pass1);
  long long L = 0, NB = 0;
  for (int t = 0; t < T; ++t) {
    ch[t].line0 = L;
    ch[t].nb0 = NB;
    L += ch[t].lines;
    NB += ch[t].nonblank;
  }
  const long long total_lines = L;
  auto pass2 = [&](int t) {
    Chunk& c = ch[t];
    const char* p = c.b;
    long long line = c.line0, nb = c.nb0;
    auto fail = [&](long long ln, std::string msg) {
      if (c.err_line < 0) {
        c.err_line = ln;
        c.err = std::move(msg);
      }
    };
    while (p < c.e && c.err_line < 0) {
      Line l = strip(next_raw_line(p, c.e));
      ++line;
      if (l.b == l.e) continue;
      long long k = nb++;
      if (k == n_rec - 1) c.last_line = line;
      if (k == 0) continue;  // header (parsed above)
      if (k >= n_rec) {
        c.trailing = true;
        continue;
      }
      if (k <= n_obs) {
        long long o = k - 1;
        Line parts[5];
        int n = split(l, parts, 5);
        if (n != 4) {
          fail(line, "observation needs 4 fields, got " + std::to_string(n));
          break;
        }
        long long ci, pi;
        bool bc, bp;
        std::string nc_s, np_s;
        double x, y;
        if (!parse_int(parts[0], ci, bc, nc_s) || !parse_int(parts[1], pi, bp, np_s) || !parse_float(parts[2], x) ||
            !parse_float(parts[3], y)) {
          fail(line, "malformed observation " + py_repr(l));
          break;
        }
        if (bc || ci < 0 || ci >= n_cam) {
          fail(line, "camera index " + (bc ? nc_s : std::to_string(ci)) + " out of range [0, " +
                         std::to_string(n_cam) + ")");
          break;
        }
        if (bp || pi < 0 || pi >= n_pt) {
          fail(line, "point index " + (bp ? np_s : std::to_string(pi)) + " out of range [0, " +
                         std::to_string(n_pt) + ")");
          break;
        }
        cam_index[o] = ci;
        pt_index[o] = pi;
        pixels[2 * o] = x;
        pixels[2 * o + 1] = y;
        continue;
      }
      long long s = k - 1 - n_obs;
      bool is_cam = s < 9 * n_cam;
      double v;
      if (!parse_float(l, v)) {
        fail(line, "malformed float " + py_repr(l) + " in " + (is_cam ? "camera parameters" : "point coordinates"));
        break;
      }
      if (is_cam) cams[s] = v;
      else pts[s - 9 * n_cam] = v;
    }
  };
  run(pass2);
  long long best = -1;
  std::string msg;
  for (auto& c : ch)
    if (c.err_line >= 0 && (best < 0 || c.err_line < best)) {
      best = c.err_line;
      msg = c.err;
    }
  if (best >= 0) {
    set_err(best, msg, (long long*)err_line, err_msg, err_len);
    return BAMG_ERR_FORMAT;
  }
  if (NB < n_rec) {
    long long k = NB;  // first missing record
    std::string sec = (k <= n_obs) ? "observation " + std::to_string(k - 1)
                      : (k - 1 - n_obs < 9 * n_cam) ? std::string("camera parameters")
                                                    : std::string("point coordinates");
    set_err(total_lines + 1, "file ends before " + sec, (long long*)err_line, err_msg, err_len);
    return BAMG_ERR_FORMAT;
  }
  if (NB > n_rec) {
    long long last = -1;
    for (auto& c : ch)
      if (c.last_line >= 0) last = c.last_line;
    set_err(last + 1, "trailing content after point coordinates", (long long*)err_line, err_msg, err_len);
    return BAMG_ERR_FORMAT;
  }
  return 0;
}

namespace {

// f"{v:.17g}" (Python prints every NaN as "nan")
inline char* put_g17(char* o, double v) {
  if (std::isnan(v)) {
    memcpy(o, "nan", 3);
    return o + 3;
  }
  auto r = std::to_chars(o, o + 32, v, std::chars_format::general, 17);
  return r.ptr;
}

inline char* put_int(char* o, long long v) { return std::to_chars(o, o + 24, v).ptr; }

}  // namespace

extern "C" int bamg_bal_write(const char* path, int64_t n_cam, int64_t n_pt, int64_t n_obs, const int64_t* cam_index,
                              const int64_t* pt_index, const double* pixels, const double* cams, const double* pts,
                              int32_t n_threads) {
  FILE* f = fopen(path, "wb");
  if (!f) return BAMG_ERR_CUDA;
  char hdr[96];
  char* o = hdr;
  o = put_int(o, n_cam);
  *o++ = ' ';
  o = put_int(o, n_pt);
  *o++ = ' ';
  o = put_int(o, n_obs);
  *o++ = '\n';
  bool ok = fwrite(hdr, 1, (size_t)(o - hdr), f) == (size_t)(o - hdr);
  // records: n_obs observation lines, then 9 n_cam + 3 n_pt scalar lines, formatted
  // in parallel blocks and written in order
  const long long n_rec = n_obs + 9 * n_cam + 3 * n_pt;
  const long long BLK = 1 << 16;
  int T = threads_for(n_threads, (size_t)n_rec * 48);
  long long nblk = (n_rec + BLK - 1) / BLK;
  for (long long b0 = 0; b0 < nblk && ok; b0 += T) {
    int nb = (int)std::min<long long>(T, nblk - b0);
    std::vector<std::string> out(nb);
    auto fmt = [&](int t) {
      long long r0 = (b0 + t) * BLK, r1 = std::min(n_rec, r0 + BLK);
      std::string& s = out[t];
      s.resize((size_t)(r1 - r0) * 64);
      char* q = &s[0];
      for (long long r = r0; r < r1; ++r) {
        if (r < n_obs) {
          q = put_int(q, cam_index[r]);
          *q++ = ' ';
          q = put_int(q, pt_index[r]);
          *q++ = ' ';
          q = put_g17(q, pixels[2 * r]);
          *q++ = ' ';
          q = put_g17(q, pixels[2 * r + 1]);
        } else {
          long long sidx = r - n_obs;
          q = put_g17(q, sidx < 9 * n_cam ? cams[sidx] : pts[sidx - 9 * n_cam]);
        }
        *q++ = '\n';
      }
      s.resize((size_t)(q - &s[0]));
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nb; ++t) th.emplace_back(fmt, t);
    fmt(0);
    for (auto& x : th) x.join();
    for (auto& s : out)
      if (fwrite(s.data(), 1, s.size(), f) != s.size()) ok = false;
  }
  if (fclose(f) != 0) ok = false;
  return ok ? 0 : BAMG_ERR_CUDA;
}
