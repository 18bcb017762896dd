// Matrix Market ingestion: host C++ restatement of
// read_matrix_market<SR> (matrix_market.hpp:43-141) feeding the same
// normalised COO the generators return.
//
// Accepted: `%%MatrixMarket matrix coordinate {real|integer|pattern}
// {general|symmetric}` (header matched case-insensitively).  One-based file
// indices become zero-based; symmetric files mirror every off-diagonal entry;
// pattern entries take SR::one(), the others SR::from_real(value).  Then
// normalize_coo (formats.hpp:105-133): stable row-major order, duplicates
// folded with SR::add in file order, zeros dropped.
//
// Errors follow the reference: structural problems (no header, bad size
// line, wrong field count, non-numeric tokens, entries outside the declared
// dimensions, early EOF) are MalformedInputError "path:line: what"; an
// object / format / field / symmetry the reader does not handle is
// UnsupportedFormatError.  Numbers parse like std::stoll / std::stod (a
// numeric prefix is enough; no digits or out of range is an error).
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "common.cuh"
#include "semiring.cuh"

namespace spg {
namespace {

std::vector<std::string> tokens(const std::string& s) {
  std::vector<std::string> out;
  size_t i = 0;
  const size_t n = s.size();
  while (i < n) {
    while (i < n && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
    const size_t b = i;
    while (i < n && !std::isspace(static_cast<unsigned char>(s[i]))) ++i;
    if (i > b) out.emplace_back(s, b, i - b);
  }
  return out;
}

bool parse_i64(const std::string& t, int64_t& v) {
  errno = 0;
  char* end = nullptr;
  const long long x = std::strtoll(t.c_str(), &end, 10);
  if (end == t.c_str() || errno == ERANGE) return false;
  v = x;
  return true;
}

bool parse_f64(const std::string& t, double& v) {
  errno = 0;
  char* end = nullptr;
  const double x = std::strtod(t.c_str(), &end);
  if (end == t.c_str() || errno == ERANGE) return false;
  v = x;
  return true;
}

[[noreturn]] void bad_line(const std::string& path, size_t line, const std::string& what) {
  fail(SPG_ERR_MALFORMED, path + ":" + std::to_string(line) + ": " + what);
}

template <class T>
T* hcopy(const std::vector<T>& v) {
  void* p = std::malloc(sizeof(T) * std::max<size_t>(v.size(), 1));
  if (!p) fail(SPG_ERR_OOM, "host allocation failed");
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return static_cast<T*>(p);
}

template <class SR>
void read_mm(const std::string& path, int64_t* nrows, int64_t* ncols, int64_t* nnz, int64_t** rows,
             int64_t** cols, void** vals) {
  using V = typename SR::value_type;
  std::ifstream in(path);
  if (!in) fail(SPG_ERR_MALFORMED, path + ": cannot open file");
  std::string line;
  size_t ln = 0;
  if (!std::getline(in, line)) bad_line(path, 1, "empty file");
  ++ln;
  std::string low = line;
  for (char& ch : low) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  const auto hdr = tokens(low);
  if (hdr.size() < 5 || hdr[0] != "%%matrixmarket") bad_line(path, ln, "missing %%MatrixMarket header");
  if (hdr[1] != "matrix") fail(SPG_ERR_UNSUPPORTED_FORMAT, path + ": unsupported object '" + hdr[1] + "'");
  if (hdr[2] != "coordinate")
    fail(SPG_ERR_UNSUPPORTED_FORMAT,
         path + ": unsupported format '" + hdr[2] + "' (only coordinate files are accepted)");
  const std::string& field = hdr[3];
  const bool pattern = field == "pattern";
  if (!pattern && field != "real" && field != "integer")
    fail(SPG_ERR_UNSUPPORTED_FORMAT, path + ": unsupported field '" + field + "'");
  const std::string& sym = hdr[4];
  const bool mirror = sym == "symmetric";
  if (!mirror && sym != "general")
    fail(SPG_ERR_UNSUPPORTED_FORMAT, path + ": unsupported symmetry '" + sym + "'");

  // size line: first line that is neither a comment nor blank
  std::vector<std::string> sz;
  while (sz.empty() && std::getline(in, line)) {
    ++ln;
    if (!line.empty() && line[0] == '%') continue;
    sz = tokens(line);
  }
  if (sz.size() != 3) bad_line(path, ln, "expected size line 'nrows ncols nnz'");
  int64_t m = 0, n = 0, declared = 0;
  if (!parse_i64(sz[0], m) || !parse_i64(sz[1], n) || !parse_i64(sz[2], declared))
    bad_line(path, ln, "non-numeric size line");
  if (m < 0 || n < 0 || declared < 0) bad_line(path, ln, "negative size field");

  struct Entry {
    int64_t r, c;
    V v;
  };
  std::vector<Entry> ent;
  ent.reserve(static_cast<size_t>(declared) * (mirror ? 2 : 1));
  const size_t want = pattern ? 2 : 3;
  int64_t seen = 0;
  while (seen < declared && std::getline(in, line)) {
    ++ln;
    if (!line.empty() && line[0] == '%') continue;
    const auto f = tokens(line);
    if (f.empty()) continue;
    if (f.size() != want)
      bad_line(path, ln, "expected " + std::to_string(want) + " fields, got " + std::to_string(f.size()));
    int64_t r = 0, c = 0;
    double x = 1.0;
    if (!parse_i64(f[0], r) || !parse_i64(f[1], c) || (!pattern && !parse_f64(f[2], x)))
      bad_line(path, ln, "non-numeric entry");
    if (r < 1 || r > m || c < 1 || c > n)
      bad_line(path, ln,
               "entry (" + std::to_string(r) + ", " + std::to_string(c) + ") outside declared dimensions");
    const V v = pattern ? SR::one() : SR::from_real(x);
    ent.push_back({r - 1, c - 1, v});
    if (mirror && r != c) ent.push_back({c - 1, r - 1, v});
    ++seen;
  }
  if (seen < declared)
    bad_line(path, ln, "file ends after " + std::to_string(seen) + " of " + std::to_string(declared) + " entries");

  // normalize_coo: stable row-major order, fold equal coordinates in file order, drop zeros
  std::stable_sort(ent.begin(), ent.end(),
                   [](const Entry& a, const Entry& b) { return a.r != b.r ? a.r < b.r : a.c < b.c; });
  std::vector<int64_t> orow, ocol;
  std::vector<V> oval;
  orow.reserve(ent.size());
  ocol.reserve(ent.size());
  oval.reserve(ent.size());
  for (size_t i = 0; i < ent.size();) {
    V acc = ent[i].v;
    size_t j = i + 1;
    for (; j < ent.size() && ent[j].r == ent[i].r && ent[j].c == ent[i].c; ++j) acc = SR::add(acc, ent[j].v);
    if (!SR::is_zero(acc)) {
      orow.push_back(ent[i].r);
      ocol.push_back(ent[i].c);
      oval.push_back(acc);
    }
    i = j;
  }
  *nrows = m;
  *ncols = n;
  *nnz = static_cast<int64_t>(orow.size());
  *rows = hcopy(orow);
  *cols = hcopy(ocol);
  *vals = hcopy(oval);
}

}  // namespace

void read_matrix_market(int sr, const char* path, int64_t* nrows, int64_t* ncols, int64_t* nnz, int64_t** rows,
                        int64_t** cols, void** vals) {
  const std::string p(path);
  switch (sr) {
    case SPG_SR_ARITHMETIC: read_mm<Arithmetic>(p, nrows, ncols, nnz, rows, cols, vals); break;
    case SPG_SR_MINPLUS: read_mm<MinPlus>(p, nrows, ncols, nnz, rows, cols, vals); break;
    case SPG_SR_BOOLEAN: read_mm<Boolean>(p, nrows, ncols, nnz, rows, cols, vals); break;
    case SPG_SR_MINSELECT: read_mm<MinSelect>(p, nrows, ncols, nnz, rows, cols, vals); break;
    case SPG_SR_TROPICAL_I32: read_mm<TropicalI32>(p, nrows, ncols, nnz, rows, cols, vals); break;
    case SPG_SR_MAXTIMES: read_mm<MaxTimes>(p, nrows, ncols, nnz, rows, cols, vals); break;
    default: fail(SPG_ERR_ARG, "unknown semiring id " + std::to_string(sr));
  }
}

}  // namespace spg
