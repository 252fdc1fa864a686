// Matrix Market wire format of the operator blocks: the reference's dump /
// load path for A, B and Q (proj/src/csr.cpp:126-175, written by the runner's
// --dump-matrices, proj/src/runner.cpp:223-229). A system the reference dumps
// is read here into the same CSR arrays the reference's reader would build,
// so it feeds the GPU solve unchanged (and vice versa).
//
//   write: "%%MatrixMarket matrix coordinate real general|symmetric", the
//          size line, then 1-based "i j v" lines with v at 17 significant
//          digits (std::ostream precision 17); symmetric = lower triangle only.
//   read:  same header checks and messages; symmetric off-diagonal entries
//          mirrored; triplets stably ordered by (row, col) and duplicates
//          summed from 0.0 in file order (csr_from_triplets, csr.cpp:88-111).
//
// The reader parses the whole entry list from one buffer (strtol / strtod —
// correctly rounded like the stream extraction the reference uses) and builds
// the CSR with a counting sort by row plus a stable sort of each row by
// column, which orders exactly like the reference's global stable sort.
#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "dshost.hpp"

namespace dshost {

void write_matrix_market(const Csr& a, const std::string& path, bool symmetric) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open " + path + " for writing");
  std::vector<char> buf(1 << 20);
  out.rdbuf()->pubsetbuf(buf.data(), static_cast<std::streamsize>(buf.size()));
  out << "%%MatrixMarket matrix coordinate real " << (symmetric ? "symmetric" : "general") << "\n";
  int64_t count = 0;
  for (int i = 0; i < a.n_rows; ++i)
    for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k)
      if (!symmetric || a.ci[k] <= i) ++count;
  out << a.n_rows << " " << a.n_cols << " " << count << "\n";
  out.precision(17);
  for (int i = 0; i < a.n_rows; ++i)
    for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k)
      if (!symmetric || a.ci[k] <= i) out << i + 1 << " " << a.ci[k] + 1 << " " << a.v[k] << "\n";
  out.flush();
  if (!out) throw std::runtime_error("write failed: " + path);
}

namespace {

// whitespace-separated token scanner over one buffer
struct Scan {
  const char* p;
  const char* end;
  void skip() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r' || *p == '\v' || *p == '\f')) ++p;
  }
  bool int_(long long& out) {
    skip();
    if (p >= end) return false;
    char* q = nullptr;
    errno = 0;
    out = std::strtoll(p, &q, 10);
    if (q == p || errno == ERANGE || out < INT32_MIN || out > INT32_MAX) return false;
    p = q;
    return true;
  }
  bool dbl(double& out) {
    skip();
    if (p >= end) return false;
    char* q = nullptr;
    out = std::strtod(p, &q);
    if (q == p) return false;
    // the reference's stream extraction takes decimal numbers only (no hex
    // floats, inf or nan): stop where it would
    for (const char* c = p; c < q; ++c)
      if (!((*c >= '0' && *c <= '9') || *c == '+' || *c == '-' || *c == '.' || *c == 'e' || *c == 'E')) return false;
    p = q;
    return true;
  }
};

}  // namespace

Csr read_matrix_market(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  size_t pos = 0;
  auto next_line = [&](std::string& line) {
    if (pos >= text.size()) return false;
    size_t e = text.find('\n', pos);
    if (e == std::string::npos) e = text.size();
    line.assign(text, pos, e - pos);
    pos = e + 1;
    return true;
  };
  std::string line;
  if (!next_line(line) || line.rfind("%%MatrixMarket", 0) != 0)
    throw std::runtime_error(path + ": missing MatrixMarket header");
  std::istringstream header(line);
  std::string tag, object, format, field, qualifier;
  header >> tag >> object >> format >> field >> qualifier;
  if (object != "matrix" || format != "coordinate" || field != "real")
    throw std::runtime_error(path + ": unsupported MatrixMarket type");
  const bool symmetric = qualifier == "symmetric";
  if (!symmetric && qualifier != "general") throw std::runtime_error(path + ": unsupported qualifier " + qualifier);
  bool have = false;
  while (next_line(line))
    if (!line.empty() && line[0] != '%') {
      have = true;
      break;
    }
  if (!have) line.clear();
  std::istringstream dims(line);
  int n_rows = 0, n_cols = 0;
  int64_t count = 0;
  if (!(dims >> n_rows >> n_cols >> count)) throw std::runtime_error(path + ": bad size line");
  if (n_rows < 0 || n_cols < 0 || count < 0) throw std::runtime_error(path + ": bad size line");

  // triplets in file order (mirrored symmetric entries right after their source)
  std::vector<int32_t> tr, tc;
  std::vector<double> tv;
  const size_t cap = static_cast<size_t>(symmetric ? 2 * count : count);
  tr.reserve(cap);
  tc.reserve(cap);
  tv.reserve(cap);
  Scan sc{text.data() + std::min(pos, text.size()), text.data() + text.size()};
  for (int64_t k = 0; k < count; ++k) {
    long long i = 0, j = 0;
    double v = 0.0;
    if (!sc.int_(i) || !sc.int_(j) || !sc.dbl(v)) throw std::runtime_error(path + ": truncated entry list");
    tr.push_back(static_cast<int32_t>(i - 1));
    tc.push_back(static_cast<int32_t>(j - 1));
    tv.push_back(v);
    if (symmetric && i != j) {
      tr.push_back(static_cast<int32_t>(j - 1));
      tc.push_back(static_cast<int32_t>(i - 1));
      tv.push_back(v);
    }
  }
  const size_t nt = tr.size();
  for (size_t t = 0; t < nt; ++t)
    if (tr[t] < 0 || tr[t] >= n_rows || tc[t] < 0 || tc[t] >= n_cols)
      throw std::invalid_argument("csr_from_triplets: index out of range");

  // counting sort by row (stable), then a stable sort of each row by column
  std::vector<int64_t> start(static_cast<size_t>(n_rows) + 1, 0);
  for (size_t t = 0; t < nt; ++t) ++start[tr[t] + 1];
  for (int i = 0; i < n_rows; ++i) start[i + 1] += start[i];
  std::vector<int64_t> order(nt);
  {
    std::vector<int64_t> fill(start.begin(), start.end() - 1);
    for (size_t t = 0; t < nt; ++t) order[fill[tr[t]]++] = static_cast<int64_t>(t);
  }
  Csr m;
  m.n_rows = n_rows;
  m.n_cols = n_cols;
  m.rp.assign(static_cast<size_t>(n_rows) + 1, 0);
  m.ci.reserve(nt);
  m.v.reserve(nt);
  for (int i = 0; i < n_rows; ++i) {
    auto b = order.begin() + start[i], e = order.begin() + start[i + 1];
    std::stable_sort(b, e, [&](int64_t x, int64_t y) { return tc[x] < tc[y]; });
    for (auto it = b; it != e;) {
      const int32_t col = tc[*it];
      double sum = 0.0;
      while (it != e && tc[*it] == col) sum += tv[*it++];
      m.ci.push_back(col);
      m.v.push_back(sum);
    }
    m.rp[i + 1] = static_cast<int64_t>(m.ci.size());
  }
  return m;
}

}  // namespace dshost
