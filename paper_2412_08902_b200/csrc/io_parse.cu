// Host-side ingestion (reference matrices.py:175-307 load_matrix_market / parse_edge_list):
// a multi-threaded parser of the entry lines of a Matrix Market coordinate file or of an
// edge list, feeding the CSR builders directly.  It accepts a strict subset of what the
// reference accepts (ASCII decimal tokens, the reference's comment / blank-line rules) and
// reports "irregular" for anything else, so the caller re-parses with the Python
// restatement and raises the reference's exact FormatError (message + line number).
//
//   kind 0: Matrix Market entries after the size line: E = 2 (pattern) or 3 whitespace-
//           separated tokens; row/col parsed as floats and required integral (the
//           reference's numpy fast path), values with strtod (correctly rounded, as numpy);
//           lines that strip to '' or start with '%' are skipped.
//   kind 1: edge list 'u v' (',' also separates), ids [+-]?[0-9]+; lines that strip to ''
//           or start with '#' / '%' are skipped.
// The file is split into byte ranges on line boundaries; pass 1 counts data lines per range,
// pass 2 parses each range into its slice of the output (file order preserved).
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fcntl.h>
#include <locale.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <thread>
#include <unistd.h>
#include <vector>

#include "common.cuh"

namespace {

enum { kOk = 0, kIrregular = 1 };

locale_t c_numeric() {  // strtod must not follow the process locale
  static locale_t l = newlocale(LC_NUMERIC_MASK, "C", (locale_t)0);
  return l;
}

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\f' || c == '\v'; }

struct Mapped {
  const char* p = nullptr;
  size_t n = 0;
  int fd = -1;
  ~Mapped() {
    if (p && n) munmap(const_cast<char*>(p), n);
    if (fd >= 0) close(fd);
  }
};

// [b, e) of the stripped line starting at s (s < end); returns the next line start
inline const char* next_line(const char* s, const char* end, const char*& b, const char*& e) {
  const char* nl = static_cast<const char*>(memchr(s, '\n', (size_t)(end - s)));
  const char* le = nl ? nl : end;
  b = s;
  e = le;
  while (b < e && is_space(*b)) ++b;
  while (e > b && is_space(e[-1])) --e;
  return nl ? nl + 1 : end;
}

inline bool skipped(const char* b, const char* e, int kind) {
  return b == e || *b == '%' || (kind == 1 && *b == '#');
}

// strict decimal float token [+-]?(d+(.d*)?|.d+)([eE][+-]?d+)?
inline bool float_token(const char* b, const char* e, double& out) {
  const char* q = b;
  if (q < e && (*q == '+' || *q == '-')) ++q;
  int digits = 0;
  while (q < e && *q >= '0' && *q <= '9') ++q, ++digits;
  if (q < e && *q == '.') {
    ++q;
    while (q < e && *q >= '0' && *q <= '9') ++q, ++digits;
  }
  if (!digits) return false;
  if (q < e && (*q == 'e' || *q == 'E')) {
    ++q;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    int ed = 0;
    while (q < e && *q >= '0' && *q <= '9') ++q, ++ed;
    if (!ed) return false;
  }
  if (q != e || e - b > 300) return false;
  char buf[320];
  memcpy(buf, b, (size_t)(e - b));
  buf[e - b] = 0;
  errno = 0;
  out = strtod_l(buf, nullptr, c_numeric());
  return errno != ERANGE || out != 0.0;  // underflow to 0 is the reference's value too; overflow -> inf kept
}

inline bool int_token(const char* b, const char* e, int64_t& out) {
  const char* q = b;
  bool neg = false;
  if (q < e && (*q == '+' || *q == '-')) neg = *q++ == '-';
  if (q == e || e - q > 18) return false;
  int64_t v = 0;
  for (; q < e; ++q) {
    if (*q < '0' || *q > '9') return false;
    v = v * 10 + (*q - '0');
  }
  out = neg ? -v : v;
  return true;
}

// split [b, e) into up to `cap` tokens on whitespace (and ',' for edge lists)
inline int tokens(const char* b, const char* e, int kind, const char** tb, const char** te, int cap) {
  int n = 0;
  const char* q = b;
  while (q < e) {
    while (q < e && (is_space(*q) || (kind == 1 && *q == ','))) ++q;
    if (q == e) break;
    const char* s = q;
    while (q < e && !is_space(*q) && !(kind == 1 && *q == ',')) ++q;
    if (n == cap) return cap + 1;
    tb[n] = s;
    te[n] = q;
    ++n;
  }
  return n;
}

struct Range {
  const char* b;
  const char* e;
  int64_t count = 0;
  int status = kOk;
};

std::vector<Range> split_ranges(const char* p, size_t n, int parts) {
  std::vector<Range> r;
  const char* end = p + n;
  const char* s = p;
  for (int i = 0; i < parts && s < end; ++i) {
    const char* t = (i == parts - 1) ? end : p + (size_t)((double)n * (i + 1) / parts);
    if (t < s) t = s;
    if (t < end) {
      const char* nl = static_cast<const char*>(memchr(t, '\n', (size_t)(end - t)));
      t = nl ? nl + 1 : end;
    }
    r.push_back({s, t});
    s = t;
  }
  return r;
}

bool open_map(const char* path, Mapped& m) {
  m.fd = open(path, O_RDONLY);
  if (m.fd < 0) return false;
  struct stat st;
  if (fstat(m.fd, &st) != 0) return false;
  m.n = (size_t)st.st_size;
  if (m.n == 0) return true;
  void* a = mmap(nullptr, m.n, PROT_READ, MAP_PRIVATE, m.fd, 0);
  if (a == MAP_FAILED) {
    m.n = 0;
    return false;
  }
  madvise(a, m.n, MADV_SEQUENTIAL);
  m.p = static_cast<const char*>(a);
  return true;
}

int parse_range(Range& rg, int kind, int expected, int64_t* a, int64_t* b, double* v, bool write) {
  const char* s = rg.b;
  int64_t k = 0;
  const char* tb[4];
  const char* te[4];
  while (s < rg.e) {
    const char *lb, *le;
    s = next_line(s, rg.e, lb, le);
    if (skipped(lb, le, kind)) continue;
    for (const char* q = lb; q < le; ++q)  // non-ASCII / control bytes: leave to the reference rules
      if ((unsigned char)*q >= 0x80 || ((unsigned char)*q < 0x20 && !is_space(*q))) return kIrregular;
    if (write) {
      if (tokens(lb, le, kind, tb, te, 3) != expected) return kIrregular;
      if (kind == 1) {
        int64_t u, w;
        if (!int_token(tb[0], te[0], u) || !int_token(tb[1], te[1], w) || u < 0 || w < 0) return kIrregular;
        a[k] = u;
        b[k] = w;
      } else {
        double i, j, x = 1.0;
        if (!float_token(tb[0], te[0], i) || !float_token(tb[1], te[1], j)) return kIrregular;
        if (i != std::floor(i) || j != std::floor(j) || std::fabs(i) > 9e15 || std::fabs(j) > 9e15) return kIrregular;
        if (expected == 3 && !float_token(tb[2], te[2], x)) return kIrregular;
        a[k] = (int64_t)i;
        b[k] = (int64_t)j;
        v[k] = x;
      }
    }
    ++k;
  }
  rg.count = k;
  return kOk;
}

}  // namespace

extern "C" {

// Number of data (entry) lines of `path` from byte `offset` (kind 0: Matrix Market entries,
// 1: edge list).  Status HCS_OK; *irregular = 1 when a line needs the reference's rules.
int hcs_io_count(const char* path, int64_t offset, int kind, int nthreads, int64_t* count, int* irregular) {
  HCS_REQUIRE(path && count && irregular && offset >= 0 && (kind == 0 || kind == 1), HCS_EINVAL, "bad arguments");
  Mapped m;
  HCS_REQUIRE(open_map(path, m), HCS_EINVAL, "cannot map %s", path);
  *count = 0;
  *irregular = 0;
  if ((size_t)offset >= m.n) return HCS_OK;
  const int parts = nthreads > 0 ? nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
  auto rs = split_ranges(m.p + offset, m.n - (size_t)offset, parts);
  std::vector<std::thread> th;
  for (auto& r : rs) th.emplace_back([&r, kind] { r.status = parse_range(r, kind, 0, nullptr, nullptr, nullptr, false); });
  for (auto& t : th) t.join();
  for (auto& r : rs) {
    if (r.status != kOk) *irregular = 1;
    *count += r.count;
  }
  return HCS_OK;
}

// Parse the data lines into a[i], b[i] (row/col as written, or u/v) and v[i] (kind 0 with
// expected = 3; 1.0 otherwise).  `count` must be hcs_io_count's result.  *irregular = 1 ->
// outputs unusable, re-parse with the reference rules.
int hcs_io_parse(const char* path, int64_t offset, int kind, int expected, int64_t count, int nthreads, int64_t* a,
                 int64_t* b, double* v, int* irregular) {
  HCS_REQUIRE(path && a && b && irregular && offset >= 0 && (kind == 0 || kind == 1), HCS_EINVAL, "bad arguments");
  HCS_REQUIRE(kind == 1 ? expected == 2 : (expected == 2 || expected == 3), HCS_EINVAL, "bad field count");
  HCS_REQUIRE(kind == 1 || v, HCS_EINVAL, "values buffer required");
  Mapped m;
  HCS_REQUIRE(open_map(path, m), HCS_EINVAL, "cannot map %s", path);
  *irregular = 0;
  if ((size_t)offset >= m.n) {
    *irregular = count != 0;
    return HCS_OK;
  }
  const int parts = nthreads > 0 ? nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
  auto rs = split_ranges(m.p + offset, m.n - (size_t)offset, parts);
  std::vector<std::thread> th;
  for (auto& r : rs) th.emplace_back([&r, kind] { r.status = parse_range(r, kind, 0, nullptr, nullptr, nullptr, false); });
  for (auto& t : th) t.join();
  std::vector<int64_t> base(rs.size() + 1, 0);
  for (size_t i = 0; i < rs.size(); ++i) {
    if (rs[i].status != kOk) *irregular = 1;
    base[i + 1] = base[i] + rs[i].count;
  }
  if (*irregular || base.back() != count) {
    *irregular = 1;
    return HCS_OK;
  }
  th.clear();
  for (size_t i = 0; i < rs.size(); ++i)
    th.emplace_back([&, i] {
      rs[i].status = parse_range(rs[i], kind, expected, a + base[i], b + base[i], v ? v + base[i] : nullptr, true);
    });
  for (auto& t : th) t.join();
  for (auto& r : rs)
    if (r.status != kOk) *irregular = 1;
  if (kind == 0 && expected == 2)
    for (int64_t i = 0; i < count; ++i) v[i] = 1.0;
  return HCS_OK;
}

}  // extern "C"
