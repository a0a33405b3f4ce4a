// Graph file loaders: load_graph (graph.cpp:68-161, 180-184) restated
// over the C ABI — MatrixMarket coordinate files (pattern / real / integer, general /
// symmetric, 1-based) and whitespace edge lists (`u v [w]`, `#` / `%` comments, a
// `% vertices N` declaration). Same accepted inputs, same error messages and the same
// error kinds (FormatError -> NULPA_EFORMAT, ValidationError -> NULPA_EINVAL). Parsing is
// host I/O; the CSR is then built on the device (build_csr.cu).
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <string_view>
#include <vector>

#include "internal.hpp"

namespace nulpa {

nulpa_graph* build_csr_device(const uint32_t* u, const uint32_t* v, const double* w, uint64_t ne,
                              int64_t n_declared, int symmetrize, int device);

namespace {

constexpr uint64_t kMaxVertexId = 0xFFFFFFFEull;  // 0xFFFFFFFF is reserved (graph.cpp:18)

struct Parsed {
  std::vector<uint32_t> u, v;
  std::vector<double> w;
  int64_t n_declared = -1;
};

[[noreturn]] void format_fail(const std::string& path, size_t line, const std::string& what) {
  throw Error(NULPA_EFORMAT, path + ":" + std::to_string(line) + ": " + what);
}

std::vector<std::string_view> split_ws(std::string_view s) {
  std::vector<std::string_view> out;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
    size_t j = i;
    while (j < s.size() && !std::isspace(static_cast<unsigned char>(s[j]))) ++j;
    if (j > i) out.push_back(s.substr(i, j - i));
    i = j;
  }
  return out;
}

uint64_t parse_id(std::string_view tok, const std::string& path, size_t line) {
  uint64_t v = 0;
  auto [p, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (ec != std::errc() || p != tok.data() + tok.size())
    format_fail(path, line, "expected a vertex id, got '" + std::string(tok) + "'");
  return v;
}

double parse_weight(std::string_view tok, const std::string& path, size_t line) {
  double w = 0;
  auto [p, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), w);
  if (ec != std::errc() || p != tok.data() + tok.size())
    format_fail(path, line, "expected a weight, got '" + std::string(tok) + "'");
  if (!std::isfinite(w) || w <= 0.0)
    throw Error(NULPA_EINVAL, path + ":" + std::to_string(line) +
                                  ": weight must be finite and > 0, got " + std::string(tok));
  return w;
}

void check_id_range(uint64_t id, const std::string& path, size_t line) {
  if (id > kMaxVertexId)
    throw Error(NULPA_EINVAL, path + ":" + std::to_string(line) + ": vertex id " +
                                  std::to_string(id) + " exceeds the 32-bit id space");
}

std::string lower(std::string_view s) {
  std::string out(s);
  for (char& c : out) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return out;
}

void push(Parsed& el, uint64_t a, uint64_t b, double w) {
  el.u.push_back(static_cast<uint32_t>(a));
  el.v.push_back(static_cast<uint32_t>(b));
  el.w.push_back(w);
}

// graph.cpp:68-130
Parsed load_matrix_market(std::ifstream& in, const std::string& path) {
  Parsed el;
  std::string buf;
  size_t lineno = 0;
  if (!std::getline(in, buf)) format_fail(path, 1, "empty file");
  ++lineno;
  const auto header = split_ws(buf);
  if (header.size() < 4 || lower(header[0]) != "%%matrixmarket")
    format_fail(path, lineno, "missing %%MatrixMarket banner");
  if (lower(header[1]) != "matrix" || lower(header[2]) != "coordinate")
    format_fail(path, lineno, "only 'matrix coordinate' files are supported");
  const std::string field = lower(header[3]);
  if (field != "real" && field != "integer" && field != "pattern")
    format_fail(path, lineno, "unsupported field '" + field + "' (need real, integer or pattern)");
  const std::string symmetry = header.size() >= 5 ? lower(header[4]) : "general";
  if (symmetry != "general" && symmetry != "symmetric")
    format_fail(path, lineno,
                "unsupported symmetry '" + symmetry + "' (need general or symmetric)");
  uint64_t rows = 0, cols = 0, nnz = 0;
  for (;;) {  // size line: first non-comment, non-blank line after the banner
    if (!std::getline(in, buf)) format_fail(path, lineno + 1, "missing size line");
    ++lineno;
    const auto t = split_ws(buf);
    if (t.empty() || t[0][0] == '%') continue;
    if (t.size() != 3) format_fail(path, lineno, "size line must be 'rows cols nnz'");
    rows = parse_id(t[0], path, lineno);
    cols = parse_id(t[1], path, lineno);
    nnz = parse_id(t[2], path, lineno);
    break;
  }
  const uint64_t n = std::max(rows, cols);
  if (n > kMaxVertexId + 1)
    throw Error(NULPA_EINVAL, path + ": declared dimension exceeds the 32-bit id space");
  el.n_declared = static_cast<int64_t>(n);
  el.u.reserve(nnz);
  el.v.reserve(nnz);
  el.w.reserve(nnz);
  const size_t want = field == "pattern" ? 2 : 3;
  for (uint64_t seen = 0; seen < nnz;) {
    if (!std::getline(in, buf))
      format_fail(path, lineno + 1, "unexpected end of file: expected " + std::to_string(nnz) +
                                        " entries, got " + std::to_string(seen));
    ++lineno;
    const auto t = split_ws(buf);
    if (t.empty() || t[0][0] == '%') continue;
    if (t.size() != want)
      format_fail(path, lineno, "expected " + std::to_string(want) + " tokens per entry");
    const uint64_t i = parse_id(t[0], path, lineno);
    const uint64_t j = parse_id(t[1], path, lineno);
    if (i == 0 || j == 0) format_fail(path, lineno, "MatrixMarket indices are 1-based");
    if (i > rows || j > cols)
      throw Error(NULPA_EINVAL, path + ":" + std::to_string(lineno) + ": entry (" +
                                    std::to_string(i) + "," + std::to_string(j) +
                                    ") outside declared " + std::to_string(rows) + "x" +
                                    std::to_string(cols));
    const double w = field == "pattern" ? 1.0 : parse_weight(t[2], path, lineno);
    push(el, i - 1, j - 1, w);
    ++seen;
  }
  return el;
}

// graph.cpp:132-161
Parsed load_edge_list(std::ifstream& in, const std::string& path) {
  Parsed el;
  std::string buf;
  size_t lineno = 0;
  while (std::getline(in, buf)) {
    ++lineno;
    const auto t = split_ws(buf);
    if (t.empty() || t[0][0] == '#' || t[0][0] == '%') {
      // `% vertices N` (or `# vertices N`) declares the vertex count
      if (t.size() == 3 && (t[0] == "%" || t[0] == "#") && t[1] == "vertices") {
        const uint64_t n = parse_id(t[2], path, lineno);
        if (n > kMaxVertexId + 1)
          throw Error(NULPA_EINVAL, path + ":" + std::to_string(lineno) +
                                        ": declared vertex count exceeds the 32-bit id space");
        el.n_declared = static_cast<int64_t>(n);
      }
      continue;
    }
    if (t.size() != 2 && t.size() != 3) format_fail(path, lineno, "expected 'u v' or 'u v w'");
    const uint64_t a = parse_id(t[0], path, lineno);
    const uint64_t b = parse_id(t[1], path, lineno);
    check_id_range(a, path, lineno);
    check_id_range(b, path, lineno);
    push(el, a, b, t.size() == 3 ? parse_weight(t[2], path, lineno) : 1.0);
  }
  return el;
}

Parsed load(const char* path, int format) {
  if (!path) throw Error(NULPA_EINVAL, "null path");
  if (format != NULPA_FORMAT_MATRIX_MARKET && format != NULPA_FORMAT_EDGE_LIST)
    throw Error(NULPA_EINVAL, "unknown file format");
  std::ifstream in(path);
  if (!in) throw Error(NULPA_EINVAL, std::string("cannot open input file: ") + path);
  return format == NULPA_FORMAT_MATRIX_MARKET ? load_matrix_market(in, path)
                                              : load_edge_list(in, path);
}

template <typename T>
T* copy_out(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(std::max<size_t>(1, v.size()) * sizeof(T)));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

}  // namespace
}  // namespace nulpa

using namespace nulpa;

extern "C" {

int nulpa_load_edge_list(const char* path, int format, nulpa_edge_list* out) {
  return guarded([&] {
    if (!out) throw Error(NULPA_EINVAL, "null argument");
    Parsed el = load(path, format);
    out->ne = el.u.size();
    out->n_declared = el.n_declared;
    out->u = copy_out(el.u);
    out->v = copy_out(el.v);
    out->w = copy_out(el.w);
  });
}

void nulpa_edge_list_free(nulpa_edge_list* el) {
  if (!el) return;
  std::free(el->u);
  std::free(el->v);
  std::free(el->w);
  el->u = el->v = nullptr;
  el->w = nullptr;
  el->ne = 0;
}

int nulpa_graph_load(const char* path, int format, int symmetrize, int device, nulpa_graph** out) {
  return guarded([&] {
    if (!out) throw Error(NULPA_EINVAL, "null argument");
    Parsed el = load(path, format);
    *out = build_csr_device(el.u.data(), el.v.data(), el.w.data(), el.u.size(), el.n_declared,
                            symmetrize, device);
  });
}

}  // extern "C"
