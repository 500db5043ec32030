// host_io.cpp -- STRUCTMAT / VEC / TRAJ text formats (include/parsol/io.hpp),
// byte-compatible with the reference writer (proj/src/io.cpp) and parser
// semantics (comments, ParseError / UnsupportedVersion messages with line
// numbers), but built for multi-GB files: the real lines are located once,
// then converted in parallel (OpenMP) straight into the destination vector,
// and writing formats disjoint slices in parallel.
#include <omp.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>

#include "parsol/errors.hpp"
#include "parsol/io.hpp"

namespace parsol {

std::string format_hex(double v) {
  char buf[48];
  std::snprintf(buf, sizeof buf, "%a", v);
  return buf;
}

namespace {

// Lines of a text, skipping empty lines and '#' comments; tracks line numbers.
struct Cursor {
  const char* p;
  const char* end;
  int lineno = 0;

  bool next(const char*& b, const char*& e) {
    while (p < end) {
      const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
      const char* le = nl ? nl : end;
      b = p;
      e = le;
      p = nl ? nl + 1 : end;
      ++lineno;
      if (e > b && e[-1] == '\r') --e;
      if (e == b || *b == '#') continue;
      return true;
    }
    return false;
  }
};

[[noreturn]] void parse_fail(int lineno, const std::string& what) {
  fail(Errc::ParseError, "line " + std::to_string(lineno) + ": " + what);
}

// Parse `count` reals from the cursor into out[0..count).  One sequential
// pass records where every value line starts (and each's line number); the
// conversions then run in parallel.
void parse_reals(Cursor& cur, double* out, std::size_t count, const char* what) {
  std::vector<const char*> starts(count);
  std::vector<int> lines(count);
  for (std::size_t i = 0; i < count; ++i) {
    const char *b, *e;
    if (!cur.next(b, e)) parse_fail(cur.lineno + 1, std::string("unexpected end of ") + what);
    starts[i] = b;
    lines[i] = cur.lineno;
  }
  long bad = -1;
#pragma omp parallel for schedule(static) reduction(max : bad)
  for (long i = 0; i < (long)count; ++i) {
    char* endp = nullptr;
    const double v = std::strtod(starts[i], &endp);
    if (endp == starts[i]) bad = std::max(bad, i);
    out[i] = v;
  }
  if (bad >= 0) parse_fail(lines[bad], "expected a real");
}

// format values[0..count) one per line, in parallel slices
void format_reals(std::string& out, const double* v, std::size_t count) {
  const int nt = std::max(1, omp_get_max_threads());
  std::vector<std::string> parts(nt);
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num();
    const std::size_t lo = count * t / nt, hi = count * (t + 1) / nt;
    std::string& s = parts[t];
    s.reserve((hi - lo) * 24);
    char buf[48];
    for (std::size_t i = lo; i < hi; ++i) {
      const int k = std::snprintf(buf, sizeof buf, "%a\n", v[i]);
      s.append(buf, k);
    }
  }
  std::size_t total = out.size();
  for (const auto& s : parts) total += s.size();
  out.reserve(total);
  for (const auto& s : parts) out += s;
}

}  // namespace

std::string write_matrix(const StructuredMatrix& A, const std::vector<std::string>& comments) {
  std::string out = "STRUCTMAT 1 " + std::string(kind_name(A.kind)) + ' ' + std::to_string(A.n) + ' ' +
                    std::to_string(A.m) + ' ' + std::to_string(A.s) + ' ' + std::to_string(A.r);
  if (A.kind == Kind::Babd) out += ' ' + std::to_string(A.corner_rows) + ' ' + std::to_string(A.corner_cols);
  out += '\n';
  for (const auto& c : comments) out += "# " + c + '\n';
  format_reals(out, A.data.data(), A.data.size());
  format_reals(out, A.corner.data(), A.corner.size());
  return out;
}

StructuredMatrix parse_matrix(const std::string& text) {
  Cursor cur{text.data(), text.data() + text.size()};
  const char *b, *e;
  if (!cur.next(b, e)) fail(Errc::ParseError, "empty input");
  std::istringstream hdr(std::string(b, e));
  std::string magic, kind_s;
  int version = 0, n = 0, m = 0, s = 0, r = 0;
  hdr >> magic >> version >> kind_s >> n >> m >> s >> r;
  if (magic != "STRUCTMAT" || hdr.fail()) parse_fail(cur.lineno, "bad STRUCTMAT header");
  if (version != 1) fail(Errc::UnsupportedVersion, "STRUCTMAT version " + std::to_string(version));
  const Kind kind = kind_from_name(kind_s);
  int cr = 0, cc = 0;
  if (kind == Kind::Babd) {
    hdr >> cr >> cc;
    if (hdr.fail()) parse_fail(cur.lineno, "missing corner shape");
  }
  if (n <= 0 || m <= 0) parse_fail(cur.lineno, "bad dimensions");
  std::vector<double> data(body_entry_count(kind, n, m, s, r));
  parse_reals(cur, data.data(), data.size(), "data");
  std::vector<double> corner(std::size_t(cr) * cc);
  parse_reals(cur, corner.data(), corner.size(), "corner");
  if (cur.next(b, e)) parse_fail(cur.lineno, "trailing data");
  try {
    return make(kind, n, m, s, r, std::move(data), std::move(corner), cr, cc);
  } catch (const Error& err) {
    if (err.code() == Errc::ParseError) throw;
    fail(Errc::ParseError, "invalid matrix: " + err.detail());
  }
}

std::string write_vector(const Vector& v, const std::vector<std::string>& comments) {
  std::string out = "VEC 1 " + std::to_string(v.size()) + '\n';
  for (const auto& c : comments) out += "# " + c + '\n';
  format_reals(out, v.data(), v.size());
  return out;
}

Vector parse_vector(const std::string& text) {
  Cursor cur{text.data(), text.data() + text.size()};
  const char *b, *e;
  if (!cur.next(b, e)) fail(Errc::ParseError, "empty input");
  std::istringstream hdr(std::string(b, e));
  std::string magic;
  int version = 0;
  long len = -1;
  hdr >> magic >> version >> len;
  if (magic != "VEC" || hdr.fail() || len < 0) parse_fail(cur.lineno, "bad VEC header");
  if (version != 1) fail(Errc::UnsupportedVersion, "VEC version " + std::to_string(version));
  Vector v(len);
  parse_reals(cur, v.data(), v.size(), "data");
  return v;
}

std::string write_trajectory(const Vector& flat, int m, int p, int N) {
  if ((long)flat.size() != (long)(p * N + 1) * m) fail(Errc::DimensionMismatch, "trajectory length");
  std::string out = "TRAJ 1 " + std::to_string(m) + ' ' + std::to_string(p) + ' ' + std::to_string(N) + '\n';
  format_reals(out, flat.data(), flat.size());
  return out;
}

std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) fail(Errc::IoError, "cannot open " + path);
  const std::streamsize sz = in.tellg();
  std::string s(std::size_t(sz > 0 ? sz : 0), '\0');
  in.seekg(0);
  if (sz > 0 && !in.read(s.data(), sz)) fail(Errc::IoError, "cannot read " + path);
  return s;
}

void write_file(const std::string& path, const std::string& content) {
  std::ofstream out(path, std::ios::binary);
  if (!out) fail(Errc::IoError, "cannot write " + path);
  out.write(content.data(), (std::streamsize)content.size());
  if (!out) fail(Errc::IoError, "cannot write " + path);
}

}  // namespace parsol
