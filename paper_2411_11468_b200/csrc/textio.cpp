// Text files around the hot path: graph files in, membership
// TSV in, edge lists out. Host I/O, written for throughput on billion-line files:
//
//   * the input is memory-mapped once and cut into newline-aligned chunks that are
//     tokenised by all host threads at once (no getline, no per-line std::string);
//   * every chunk stops at its first bad line; the chunks are then merged in file order,
//     so the error that surfaces — its kind, its text and its line number — is the one
//     a sequential reader would have hit first;
//   * output is formatted into per-thread byte buffers (std::to_chars) and written once.
//
// The accepted inputs, the error kinds and the message texts are the reference's,
// which callers and tests match on (FormatError -> NULPA_EFORMAT, ValidationError ->
// NULPA_EINVAL):
//   load_graph        graph.hpp:95-96, graph.cpp:68-161,180-184
//   write_edge_list   graph.hpp:112, graph.cpp:309-325
//   read_membership   io.hpp:19, io.cpp:16-56
// (write_membership formats on the device: textout.cu.)
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <optional>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace nulpa {

nulpa_graph* build_csr_device(const uint32_t* u, const uint32_t* v, const double* w, uint64_t ne,
                              int64_t n_declared, int symmetrize, int device);

namespace text {
namespace {

// Largest id a file may name: 0xFFFFFFFF is the table's empty key (graph.cpp:18).
constexpr uint64_t kIdLimit = 0xFFFFFFFEull;

// Bytes per parse chunk (NULPA_TEXT_CHUNK_BYTES overrides it: the tests cut small files
// into many chunks to exercise the in-order merge).
size_t chunk_bytes() {
  const char* e = std::getenv("NULPA_TEXT_CHUNK_BYTES");
  const long long v = e ? std::atoll(e) : 0;
  return v > 0 ? size_t(v) : size_t(8) << 20;
}

// ---- input buffer -------------------------------------------------------------------

class MappedFile {
 public:
  explicit MappedFile(const char* path) {
    fd_ = ::open(path, O_RDONLY | O_CLOEXEC);
    if (fd_ < 0) return;
    struct stat st {};
    if (::fstat(fd_, &st) != 0 || !S_ISREG(st.st_mode)) {
      ::close(fd_);
      fd_ = -1;
      return;
    }
    size_ = static_cast<size_t>(st.st_size);
    if (size_ > 0) {
      void* p = ::mmap(nullptr, size_, PROT_READ, MAP_PRIVATE, fd_, 0);
      if (p == MAP_FAILED) throw Error(NULPA_EOTHER, std::string("mmap failed: ") + path);
      ::madvise(p, size_, MADV_SEQUENTIAL | MADV_WILLNEED);
      data_ = static_cast<const char*>(p);
    }
  }
  ~MappedFile() {
    if (data_) ::munmap(const_cast<char*>(data_), size_);
    if (fd_ >= 0) ::close(fd_);
  }
  MappedFile(const MappedFile&) = delete;
  MappedFile& operator=(const MappedFile&) = delete;

  bool ok() const { return fd_ >= 0; }
  const char* begin() const { return data_; }
  const char* end() const { return data_ + size_; }

 private:
  int fd_ = -1;
  const char* data_ = nullptr;
  size_t size_ = 0;
};

// isspace() of the "C" locale, as a table.
struct SpaceTable {
  bool t[256] = {};
  constexpr SpaceTable() {
    t[uint8_t(' ')] = t[uint8_t('\t')] = t[uint8_t('\n')] = true;
    t[uint8_t('\v')] = t[uint8_t('\f')] = t[uint8_t('\r')] = true;
  }
};
constexpr SpaceTable kSpace;
inline bool space(char c) { return kSpace.t[static_cast<uint8_t>(c)]; }

// The whitespace-separated fields of one line: the first kKeep are kept, `count` keeps
// counting (a line with too many fields is an error, not a truncation).
struct Fields {
  static constexpr int kKeep = 5;
  std::string_view f[kKeep];
  int count = 0;
  bool blank() const { return count == 0; }
  bool comment(bool hash_too) const {
    return count > 0 && (f[0][0] == '%' || (hash_too && f[0][0] == '#'));
  }
};

// Walks [p, end) one '\n'-terminated line at a time (the last line may lack its '\n').
class LineCursor {
 public:
  LineCursor(const char* p, const char* end) : p_(p), end_(end) {}
  bool next(Fields& out) {
    if (p_ >= end_) return false;
    const char* nl = static_cast<const char*>(std::memchr(p_, '\n', size_t(end_ - p_)));
    const char* stop = nl ? nl : end_;
    out.count = 0;
    for (const char* c = p_; c < stop;) {
      while (c < stop && space(*c)) ++c;
      const char* s = c;
      while (c < stop && !space(*c)) ++c;
      if (c > s) {
        if (out.count < Fields::kKeep) out.f[out.count] = std::string_view(s, size_t(c - s));
        ++out.count;
      }
    }
    p_ = nl ? nl + 1 : end_;
    return true;
  }
  const char* pos() const { return p_; }

 private:
  const char* p_;
  const char* end_;
};

// ---- numbers ------------------------------------------------------------------------

// Whole-token parse; false on any leftover character, sign, overflow or empty token.
inline bool whole_u64(std::string_view t, uint64_t& v) {
  auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}
inline bool whole_f64(std::string_view t, double& v) {
  auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}

// ---- chunked parsing ----------------------------------------------------------------

// A parse failure inside a chunk: the message after "path:line: " and the chunk-local
// line number (1-based) it occurred on.
struct LineError {
  int code = NULPA_OK;
  uint64_t line = 0;
  std::string what;
  explicit operator bool() const { return code != NULPA_OK; }
};

struct Piece {
  const char* b;
  const char* e;
};

// Newline-aligned pieces of [b, e), about chunk_bytes() each, at most `cap` of them.
std::vector<Piece> split_lines(const char* b, const char* e, unsigned cap) {
  std::vector<Piece> out;
  const size_t total = size_t(e - b);
  const size_t want = std::max<size_t>(1, std::min<size_t>(cap, total / chunk_bytes() + 1));
  const size_t step = total / want + 1;
  const char* s = b;
  while (s < e) {
    const char* cut = s + std::min(step, size_t(e - s));
    if (cut < e) {
      const char* nl = static_cast<const char*>(std::memchr(cut, '\n', size_t(e - cut)));
      cut = nl ? nl + 1 : e;
    }
    out.push_back({s, cut});
    s = cut;
  }
  return out;
}

unsigned host_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return std::max(1u, std::min(h ? h : 1u, 64u));
}

// Run body(i) for i in [0, k) on up to host_threads() threads.
template <typename F>
void parallel_for(size_t k, F&& body) {
  const size_t t = std::min<size_t>(k, host_threads());
  if (t <= 1) {
    for (size_t i = 0; i < k; ++i) body(i);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(t);
  for (size_t w = 0; w < t; ++w)
    pool.emplace_back([&, w] {
      for (size_t i = w; i < k; i += t) body(i);
    });
  for (auto& th : pool) th.join();
}

unsigned max_pieces() { return std::getenv("NULPA_TEXT_CHUNK_BYTES") ? 1u << 16 : 4 * host_threads(); }

[[noreturn]] void raise_at(const std::string& path, uint64_t line, int code,
                           const std::string& what) {
  throw Error(code, path + ":" + std::to_string(line) + ": " + what);
}

// Edges parsed from one piece of a graph file.
struct EdgeChunk {
  std::vector<uint32_t> u, v;
  std::vector<double> w;
  uint64_t lines = 0;
  std::optional<uint64_t> declared;  // last `% vertices N` in the piece
  LineError err;
  void add(uint64_t a, uint64_t b, double x) {
    u.push_back(uint32_t(a));
    v.push_back(uint32_t(b));
    w.push_back(x);
  }
};

struct EdgeListOut {
  std::vector<uint32_t> u, v;
  std::vector<double> w;
  int64_t n_declared = -1;
};

void bad_id(LineError& e, uint64_t line, std::string_view tok) {
  e = {NULPA_EFORMAT, line, "expected a vertex id, got '" + std::string(tok) + "'"};
}

// A weight token: a finite float > 0 (graph.cpp:45-54).
bool weight_of(std::string_view tok, uint64_t line, double& w, LineError& e) {
  if (!whole_f64(tok, w)) {
    e = {NULPA_EFORMAT, line, "expected a weight, got '" + std::string(tok) + "'"};
    return false;
  }
  if (!std::isfinite(w) || w <= 0.0) {
    e = {NULPA_EINVAL, line, "weight must be finite and > 0, got " + std::string(tok)};
    return false;
  }
  return true;
}

// Concatenate the chunks' edges in file order (parallel copies into the final arrays).
void gather_edges(std::vector<EdgeChunk>& cs, size_t keep_chunks, uint64_t last_count,
                  EdgeListOut& out) {
  std::vector<uint64_t> at(keep_chunks + 1, 0);
  for (size_t c = 0; c < keep_chunks; ++c)
    at[c + 1] = at[c] + (c + 1 == keep_chunks ? last_count : cs[c].u.size());
  out.u.resize(at[keep_chunks]);
  out.v.resize(at[keep_chunks]);
  out.w.resize(at[keep_chunks]);
  parallel_for(keep_chunks, [&](size_t c) {
    const size_t k = at[c + 1] - at[c];
    std::copy_n(cs[c].u.begin(), k, out.u.begin() + at[c]);
    std::copy_n(cs[c].v.begin(), k, out.v.begin() + at[c]);
    std::copy_n(cs[c].w.begin(), k, out.w.begin() + at[c]);
    EdgeChunk().u.swap(cs[c].u);
    EdgeChunk().v.swap(cs[c].v);
    EdgeChunk().w.swap(cs[c].w);
  });
}

// ---- edge list: `u v [w]` lines, '#'/'%' comments, `% vertices N` (graph.cpp:132-161)

void parse_edge_piece(Piece pc, EdgeChunk& out) {
  LineCursor cur(pc.b, pc.e);
  Fields f;
  while (cur.next(f)) {
    const uint64_t line = ++out.lines;
    if (f.blank() || f.comment(true)) {
      const bool decl = f.count == 3 && (f.f[0] == "%" || f.f[0] == "#") && f.f[1] == "vertices";
      if (!decl) continue;
      uint64_t n = 0;
      if (!whole_u64(f.f[2], n)) return bad_id(out.err, line, f.f[2]);
      if (n > kIdLimit + 1) {
        out.err = {NULPA_EINVAL, line, "declared vertex count exceeds the 32-bit id space"};
        return;
      }
      out.declared = n;
      continue;
    }
    if (f.count != 2 && f.count != 3) {
      out.err = {NULPA_EFORMAT, line, "expected 'u v' or 'u v w'"};
      return;
    }
    uint64_t ends[2];
    for (int k = 0; k < 2; ++k)
      if (!whole_u64(f.f[k], ends[k])) return bad_id(out.err, line, f.f[k]);
    for (int k = 0; k < 2; ++k)
      if (ends[k] > kIdLimit) {
        out.err = {NULPA_EINVAL, line,
                   "vertex id " + std::to_string(ends[k]) + " exceeds the 32-bit id space"};
        return;
      }
    double w = 1.0;
    if (f.count == 3 && !weight_of(f.f[2], line, w, out.err)) return;
    out.add(ends[0], ends[1], w);
  }
}

EdgeListOut read_edge_list(const MappedFile& mf, const std::string& path) {
  auto pieces = split_lines(mf.begin(), mf.end(), max_pieces());
  std::vector<EdgeChunk> cs(pieces.size());
  parallel_for(pieces.size(), [&](size_t i) { parse_edge_piece(pieces[i], cs[i]); });
  EdgeListOut out;
  uint64_t base = 0;
  for (auto& c : cs) {
    if (c.err) raise_at(path, base + c.err.line, c.err.code, c.err.what);
    if (c.declared) out.n_declared = int64_t(*c.declared);
    base += c.lines;
  }
  gather_edges(cs, cs.size(), cs.empty() ? 0 : cs.back().u.size(), out);
  return out;
}

// ---- MatrixMarket coordinate (graph.cpp:68-130) -------------------------------------

struct MmHeader {
  bool pattern = false;
  uint64_t rows = 0, cols = 0, nnz = 0;
  uint64_t lines = 0;        // lines consumed through the size line
  const char* body = nullptr;  // first byte after the size line
};

std::string lowered(std::string_view s) {
  std::string r(s);
  std::transform(r.begin(), r.end(), r.begin(),
                 [](char c) { return (c >= 'A' && c <= 'Z') ? char(c - 'A' + 'a') : c; });
  return r;
}

MmHeader read_mm_header(const MappedFile& mf, const std::string& path) {
  LineCursor cur(mf.begin(), mf.end());
  Fields f;
  MmHeader h;
  auto fmt = [&](uint64_t line, const std::string& what) {
    raise_at(path, line, NULPA_EFORMAT, what);
  };
  if (!cur.next(f)) fmt(1, "empty file");
  h.lines = 1;
  // banner: %%MatrixMarket matrix coordinate <field> [<symmetry>]
  if (f.count < 4 || lowered(f.f[0]) != "%%matrixmarket") fmt(1, "missing %%MatrixMarket banner");
  if (lowered(f.f[1]) != "matrix" || lowered(f.f[2]) != "coordinate")
    fmt(1, "only 'matrix coordinate' files are supported");
  static const char* const kFields[] = {"real", "integer", "pattern"};
  const std::string field = lowered(f.f[3]);
  if (std::none_of(std::begin(kFields), std::end(kFields), [&](const char* k) { return field == k; }))
    fmt(1, "unsupported field '" + field + "' (need real, integer or pattern)");
  h.pattern = field == "pattern";
  // symmetric files list one triangle; build_csr's symmetrize adds the mirror
  const std::string sym = f.count >= 5 ? lowered(f.f[4]) : std::string("general");
  if (sym != "general" && sym != "symmetric")
    fmt(1, "unsupported symmetry '" + sym + "' (need general or symmetric)");
  for (;;) {
    if (!cur.next(f)) fmt(h.lines + 1, "missing size line");
    ++h.lines;
    if (f.blank() || f.comment(false)) continue;
    if (f.count != 3) fmt(h.lines, "size line must be 'rows cols nnz'");
    uint64_t* dst[3] = {&h.rows, &h.cols, &h.nnz};
    for (int k = 0; k < 3; ++k)
      if (!whole_u64(f.f[k], *dst[k]))
        fmt(h.lines, "expected a vertex id, got '" + std::string(f.f[k]) + "'");
    break;
  }
  if (std::max(h.rows, h.cols) > kIdLimit + 1)
    throw Error(NULPA_EINVAL, path + ": declared dimension exceeds the 32-bit id space");
  h.body = cur.pos();
  return h;
}

void parse_mm_piece(Piece pc, const MmHeader& h, EdgeChunk& out) {
  LineCursor cur(pc.b, pc.e);
  Fields f;
  const int want = h.pattern ? 2 : 3;
  while (cur.next(f)) {
    const uint64_t line = ++out.lines;
    if (f.blank() || f.comment(false)) continue;
    if (f.count != want) {
      out.err = {NULPA_EFORMAT, line, "expected " + std::to_string(want) + " tokens per entry"};
      return;
    }
    uint64_t ij[2];
    for (int k = 0; k < 2; ++k)
      if (!whole_u64(f.f[k], ij[k])) return bad_id(out.err, line, f.f[k]);
    if (ij[0] == 0 || ij[1] == 0) {
      out.err = {NULPA_EFORMAT, line, "MatrixMarket indices are 1-based"};
      return;
    }
    if (ij[0] > h.rows || ij[1] > h.cols) {
      out.err = {NULPA_EINVAL, line,
                 "entry (" + std::to_string(ij[0]) + "," + std::to_string(ij[1]) +
                     ") outside declared " + std::to_string(h.rows) + "x" + std::to_string(h.cols)};
      return;
    }
    double w = 1.0;
    if (!h.pattern && !weight_of(f.f[2], line, w, out.err)) return;
    out.add(ij[0] - 1, ij[1] - 1, w);
  }
}

EdgeListOut read_matrix_market(const MappedFile& mf, const std::string& path) {
  const MmHeader h = read_mm_header(mf, path);
  auto pieces = split_lines(h.body, mf.end(), max_pieces());
  std::vector<EdgeChunk> cs(pieces.size());
  parallel_for(pieces.size(), [&](size_t i) { parse_mm_piece(pieces[i], h, cs[i]); });
  // A sequential reader stops after the nnz-th entry: whatever follows it, bad lines
  // included, is never read. A chunk's error therefore only counts when it comes
  // before entry nnz.
  EdgeListOut out;
  out.n_declared = int64_t(std::max(h.rows, h.cols));
  uint64_t base = h.lines, seen = 0;
  size_t c = 0;
  for (; c < cs.size(); ++c) {
    const uint64_t k = cs[c].u.size();
    if (seen + k >= h.nnz) {  // entry nnz lies in this chunk: stop here
      gather_edges(cs, c + 1, h.nnz - seen, out);
      return out;
    }
    if (cs[c].err) raise_at(path, base + cs[c].err.line, cs[c].err.code, cs[c].err.what);
    seen += k;
    base += cs[c].lines;
  }
  if (h.nnz == 0) {
    gather_edges(cs, 0, 0, out);
    return out;
  }
  raise_at(path, base + 1, NULPA_EFORMAT,
           "unexpected end of file: expected " + std::to_string(h.nnz) + " entries, got " +
               std::to_string(seen));
}

EdgeListOut read_graph_file(const char* path, int format) {
  if (!path) throw Error(NULPA_EINVAL, "null path");
  if (format != NULPA_FORMAT_MATRIX_MARKET && format != NULPA_FORMAT_EDGE_LIST)
    throw Error(NULPA_EINVAL, "unknown file format");
  MappedFile mf(path);
  if (!mf.ok()) throw Error(NULPA_EINVAL, std::string("cannot open input file: ") + path);
  return format == NULPA_FORMAT_MATRIX_MARKET ? read_matrix_market(mf, path)
                                              : read_edge_list(mf, path);
}

// ---- membership TSV: `vertex<TAB>label` (io.cpp:16-56) ------------------------------

struct Assignment {
  uint32_t vertex, label;
  uint32_t line;  // chunk-local
};

struct MembershipChunk {
  std::vector<Assignment> rows;
  uint64_t lines = 0;
  LineError err;           // format error (stops the chunk)
  LineError first_range;   // first id >= n in the chunk, with its position
  size_t first_range_at = SIZE_MAX;
};

void parse_membership_piece(Piece pc, uint64_t n, MembershipChunk& out) {
  LineCursor cur(pc.b, pc.e);
  Fields f;
  while (cur.next(f)) {
    const uint64_t line = ++out.lines;
    if (f.blank() || f.comment(true)) continue;
    // field 1 must be a whole number; field 2 a number, possibly followed by junk
    // ("trailing content"), and nothing may follow it.
    uint64_t vertex = 0, label = 0;
    bool ok = whole_u64(f.f[0], vertex) && f.count >= 2;
    const char* stop = nullptr;
    if (ok) {
      auto r = std::from_chars(f.f[1].data(), f.f[1].data() + f.f[1].size(), label);
      ok = r.ec == std::errc() && r.ptr != f.f[1].data();
      stop = r.ptr;
    }
    if (!ok) {
      out.err = {NULPA_EFORMAT, line, "expected 'vertex<TAB>label'"};
      return;
    }
    if (f.count > 2 || stop != f.f[1].data() + f.f[1].size()) {
      out.err = {NULPA_EFORMAT, line, "trailing content after label"};
      return;
    }
    if ((vertex >= n || label >= n) && out.first_range_at == SIZE_MAX) {
      out.first_range_at = out.rows.size();
      out.first_range = {NULPA_EINVAL, line,
                         vertex >= n ? "vertex " + std::to_string(vertex) + " out of range for n=" +
                                           std::to_string(n)
                                     : "label " + std::to_string(label) + " out of range for n=" +
                                           std::to_string(n)};
      return;  // nothing after it can surface first
    }
    out.rows.push_back({uint32_t(vertex), uint32_t(label), uint32_t(line)});
  }
}

void read_membership_file(const char* path, uint32_t n, uint32_t* labels) {
  MappedFile mf(path);
  if (!mf.ok()) throw Error(NULPA_EINVAL, std::string("cannot open membership file: ") + path);
  auto pieces = split_lines(mf.begin(), mf.end(), max_pieces());
  std::vector<MembershipChunk> cs(pieces.size());
  parallel_for(pieces.size(), [&](size_t i) { parse_membership_piece(pieces[i], n, cs[i]); });
  std::vector<uint8_t> seen(n, 0);
  std::fill_n(labels, n, 0u);
  uint64_t base = 0;
  for (auto& c : cs) {
    for (const Assignment& a : c.rows) {
      if (seen[a.vertex])
        raise_at(path, base + a.line, NULPA_EINVAL,
                 "vertex " + std::to_string(a.vertex) + " assigned twice");
      seen[a.vertex] = 1;
      labels[a.vertex] = a.label;
    }
    if (c.first_range_at != SIZE_MAX)
      raise_at(path, base + c.first_range.line, c.first_range.code, c.first_range.what);
    if (c.err) raise_at(path, base + c.err.line, c.err.code, c.err.what);
    base += c.lines;
  }
  const auto hole = std::find(seen.begin(), seen.end(), uint8_t(0));
  if (hole != seen.end())
    throw Error(NULPA_EINVAL, std::string(path) + ": no label for vertex " +
                                  std::to_string(hole - seen.begin()));
}

// ---- edge list out (graph.cpp:309-325) ---------------------------------------------

// Each undirected edge once as `u v w` with u <= v (self-loops included), rows in order,
// w in the shortest form that reads back as the same float.
void write_edges(const char* path, const nulpa_csr* g) {
  std::FILE* fp = std::fopen(path, "wb");
  if (!fp) throw Error(NULPA_EINVAL, std::string("cannot open output file: ") + path);
  std::string head = "% undirected weighted edge list: u v w (each edge once, u <= v)\n% vertices " +
                     std::to_string(g->n) + "\n";
  bool good = std::fwrite(head.data(), 1, head.size(), fp) == head.size();
  // rows cut into ~equal edge ranges, each formatted by one thread into its own buffer
  const uint64_t n = g->n;
  const unsigned parts =
      unsigned(std::min<uint64_t>(uint64_t(host_threads()) * 4, g->m2 / (1u << 20) + 1));
  std::vector<uint64_t> cut(parts + 1, n);
  cut[0] = 0;
  for (unsigned p = 1; p < parts; ++p)
    cut[p] = uint64_t(std::upper_bound(g->offsets, g->offsets + n + 1, g->m2 * p / parts) -
                      g->offsets) - 1;
  for (unsigned p = 1; p <= parts; ++p) cut[p] = std::max(cut[p], cut[p - 1]);
  const unsigned wave = host_threads();
  std::vector<std::string> buf(wave);
  for (unsigned p0 = 0; p0 < parts && good; p0 += wave) {
    const unsigned k = std::min(wave, parts - p0);
    parallel_for(k, [&](size_t t) {
      std::string& s = buf[t];
      s.clear();
      char num[48];
      for (uint64_t i = cut[p0 + t]; i < cut[p0 + t + 1]; ++i) {
        for (uint64_t e = g->offsets[i]; e < g->offsets[i + 1]; ++e) {
          const uint32_t j = g->targets[e];
          if (j < i) continue;
          char* q = std::to_chars(num, num + sizeof num, uint32_t(i)).ptr;
          *q++ = ' ';
          q = std::to_chars(q, num + sizeof num, j).ptr;
          *q++ = ' ';
          q = std::to_chars(q, num + sizeof num, g->weights ? g->weights[e] : 1.0f).ptr;
          *q++ = '\n';
          s.append(num, size_t(q - num));
        }
      }
    });
    for (unsigned t = 0; t < k && good; ++t)
      good = std::fwrite(buf[t].data(), 1, buf[t].size(), fp) == buf[t].size();
  }
  good = (std::fclose(fp) == 0) && good;
  if (!good) throw Error(NULPA_EINVAL, std::string("failed writing ") + path);
}

template <typename T>
T* malloc_copy(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(std::max<size_t>(1, v.size()) * sizeof(T)));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

}  // namespace
}  // namespace text
}  // namespace nulpa

using namespace nulpa;

extern "C" {

int nulpa_load_edge_list(const char* path, int format, nulpa_edge_list* out) {
  return guarded([&] {
    if (!out) throw Error(NULPA_EINVAL, "null argument");
    text::EdgeListOut el = text::read_graph_file(path, format);
    out->ne = el.u.size();
    out->n_declared = el.n_declared;
    out->u = text::malloc_copy(el.u);
    out->v = text::malloc_copy(el.v);
    out->w = text::malloc_copy(el.w);
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
    text::EdgeListOut el = text::read_graph_file(path, format);
    *out = build_csr_device(el.u.data(), el.v.data(), el.w.data(), el.u.size(), el.n_declared,
                            symmetrize, device);
  });
}

int nulpa_read_membership(const char* path, uint32_t n, uint32_t* labels) {
  return guarded([&] {
    if (!path || (n && !labels)) throw Error(NULPA_EINVAL, "null argument");
    text::read_membership_file(path, n, labels);
  });
}

int nulpa_write_edge_list(const char* path, const nulpa_csr* csr) {
  return guarded([&] {
    if (!path || !csr) throw Error(NULPA_EINVAL, "null argument");
    text::write_edges(path, csr);
  });
}

}  // extern "C"
