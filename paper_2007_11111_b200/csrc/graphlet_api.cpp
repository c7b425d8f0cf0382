// graphlet_api.cpp — the graphlet:: C++ API (include/graphlet/*.hpp) over the
// C-ABI (include/fglt.h). Host-side only: dictionary planning, CSR ingest and
// text parsing, conversion-matrix utilities. Every frequency is computed by
// libfglt.so on the device; there is no CPU path for the transform.
//
// Reference interfaces mirrored (proj/include/graphlet/…):
//   dictionary.hpp:29-83  Dictionary, parse_dictionary, resolve_dependencies
//   graph.hpp:41-100      SparseAdjacency, parsers, build_adjacency
//   conversion.hpp:14-61  ConversionMatrix, full_u16, sub_matrix, net_from_raw
//   kernels.hpp:105-123   TransformStats, KernelOptions, raw_frequencies
//   transform.hpp:8-23    TransformOptions, TransformResult, transform
#include <algorithm>
#include <array>
#include <charconv>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <sstream>
#include <string>

#include "fglt.h"
#include "fglt_tables.h"
#include "graphlet/transform.hpp"

namespace graphlet {

// ================================================================ dictionary
// Dictionaries are 16-bit id sets: every operation below works on the mask
// (the device plan, make_plan in fglt.cu, uses the same representation and
// the same step table, fglt_tables.h).
namespace {

// Σ16 descriptors: family order = vertex count, then edge count, then the
// degree of the incidence node (Table 1).
constexpr std::array<GraphletDescriptor, kNumGraphlets> kSigma16{{
    {0, "singleton", 1, 0, "the vertex"},
    {1, "1-path, at an end", 2, 1, "either end"},
    {2, "2-path, at an end", 3, 2, "either end"},
    {3, "bi-fork, at the root", 3, 2, "the center"},
    {4, "3-clique, at any node", 3, 3, "any vertex"},
    {5, "3-path, at an end", 4, 3, "either end"},
    {6, "3-path, at an interior node", 4, 3, "either interior vertex"},
    {7, "claw, at a leaf", 4, 3, "any leaf"},
    {8, "claw, at the root", 4, 3, "the center"},
    {9, "dipper, at the handle tip", 4, 4, "the pendant vertex"},
    {10, "dipper, at a base node", 4, 4, "either triangle vertex off the handle"},
    {11, "dipper, at the center", 4, 4, "the degree-3 vertex"},
    {12, "4-cycle, at any node", 4, 4, "any vertex"},
    {13, "diamond, at an off-cord node", 4, 5, "either degree-2 vertex"},
    {14, "diamond, at an on-cord node", 4, 5, "either degree-3 vertex"},
    {15, "4-clique, at any node", 4, 6, "any vertex"},
}};

constexpr std::uint32_t kMandatory = 0x3u;  // {0, 1} are always members

[[noreturn]] void id_out_of_range(long long id) {
  throw ParseError("graphlet id " + std::to_string(id) + " outside 0..15");
}

std::vector<int> ids_of_mask(std::uint32_t m) {
  std::vector<int> out;
  for (int id = 0; m; ++id, m >>= 1)
    if (m & 1u) out.push_back(id);
  return out;
}

// Blanks (spaces only, as in the reference grammar) off both ends.
std::string_view trim_blanks(std::string_view s) {
  const std::size_t b = s.find_first_not_of(' ');
  if (b == std::string_view::npos) return {};
  return s.substr(b, s.find_last_not_of(' ') - b + 1);
}

// One graphlet id token: an optionally signed decimal filling the whole token
// (what std::from_chars<int> accepts: '-' allowed, '+' not).
int parse_id(std::string_view tok) {
  const bool neg = !tok.empty() && tok.front() == '-';
  const std::string_view digits = tok.substr(neg ? 1 : 0);
  long long v = 0;
  bool ok = !digits.empty();
  for (char ch : digits) {
    ok = ok && ch >= '0' && ch <= '9' && v <= (1ll << 31);
    if (ok) v = v * 10 + (ch - '0');
  }
  if (ok && !neg && v > 0x7fffffffll) ok = false;          // int overflow: from_chars fails too
  if (ok && neg && v > 0x80000000ll) ok = false;
  if (!ok) throw ParseError("malformed graphlet id '" + std::string(tok) + "'");
  if (neg ? v != 0 : v >= kNumGraphlets) id_out_of_range(neg ? -v : v);
  return static_cast<int>(v);
}

// Ids named by one comma-separated item: "k" or "lo-hi" (inclusive).
std::uint32_t item_mask(std::string_view item) {
  const std::size_t dash = item.find('-');
  if (dash == std::string_view::npos) return 1u << parse_id(item);
  const int lo = parse_id(trim_blanks(item.substr(0, dash)));
  const int hi = parse_id(trim_blanks(item.substr(dash + 1)));
  if (hi < lo) throw ParseError("descending range '" + std::string(item) + "' in dictionary spec");
  return ((2u << hi) - 1u) & ~((1u << lo) - 1u);
}

}  // namespace

std::span<const GraphletDescriptor, kNumGraphlets> graphlet_descriptors() { return kSigma16; }

Dictionary Dictionary::from_ids(std::span<const int> ids) {
  std::uint32_t m = kMandatory;
  for (int id : ids) {
    if (id < 0 || id >= kNumGraphlets) id_out_of_range(id);
    m |= 1u << id;
  }
  Dictionary d;
  d.ids_ = ids_of_mask(m);
  return d;
}

Dictionary Dictionary::all() {
  Dictionary d;
  d.ids_ = ids_of_mask((1u << kNumGraphlets) - 1u);
  return d;
}

bool Dictionary::contains(int id) const { return id >= 0 && id < kNumGraphlets && (mask() >> id & 1u); }

std::size_t Dictionary::position_of(int id) const {
  if (!contains(id)) throw Error("graphlet " + std::to_string(id) + " not in dictionary");
  // members below id, i.e. the popcount of the mask under bit id
  return static_cast<std::size_t>(__builtin_popcount(mask() & ((1u << id) - 1u)));
}

std::uint32_t Dictionary::mask() const {
  std::uint32_t m = 0;
  for (int id : ids_) m |= 1u << id;
  return m;
}

// Grammar (the reference's, proj/src/dictionary.cpp): "all", or comma-
// separated items "k" / "lo-hi" with blanks allowed around items and dashes.
// Items are checked left to right, so the first bad item decides the error.
ParsedDictionary parse_dictionary(std::string_view spec) {
  spec = trim_blanks(spec);
  if (spec.empty()) throw ParseError("empty dictionary spec");
  std::uint32_t named = 0;
  if (spec == "all") {
    named = (1u << kNumGraphlets) - 1u;
  } else {
    std::vector<std::string_view> items;
    for (std::size_t at = 0;;) {
      const std::size_t comma = std::min(spec.find(',', at), spec.size());
      items.push_back(spec.substr(at, comma - at));
      if (comma == spec.size()) break;
      at = comma + 1;
    }
    for (std::size_t i = 0; i < items.size(); ++i) {
      if (i + 1 == items.size() && i > 0 && items[i].empty())
        throw ParseError("trailing comma in dictionary spec");
      const std::string_view item = trim_blanks(items[i]);
      if (item.empty()) throw ParseError("empty token in dictionary spec");
      named |= item_mask(item);
    }
  }
  ParsedDictionary out;
  const std::vector<int> ids = ids_of_mask(named);
  out.dict = Dictionary::from_ids(std::span<const int>(ids.data(), ids.size()));
  out.implicitly_added = ids_of_mask(kMandatory & ~named);
  return out;
}

const char* aux_step_name(AuxStep s) {
  const int i = static_cast<int>(s);
  return i >= 0 && i < fglt_tables::kNumAuxSteps ? fglt_tables::kAuxSteps[i].name : "?";
}

std::vector<AuxStep> resolve_dependencies(const Dictionary& d) {
  std::vector<AuxStep> plan;
  for (int i = 0; i < fglt_tables::kNumAuxSteps; ++i)
    if (d.mask() & fglt_tables::kAuxSteps[i].needed_by) plan.push_back(static_cast<AuxStep>(i));
  return plan;
}

// A member's net count is exact only if every graphlet it is a subgraph of
// (U16 row entries right of the diagonal) is selected too.
std::vector<FamilyAdvisory> warn_incomplete_family(const Dictionary& d) {
  std::vector<FamilyAdvisory> out;
  const std::uint32_t have = d.mask();
  for (int id : d.ids()) {
    std::uint32_t need = 0;
    for (int c = id + 1; c < kNumGraphlets; ++c)
      if (fglt_tables::u16_coef(id, c)) need |= 1u << c;
    const std::uint32_t missing = need & ~have;
    if (!missing) continue;
    FamilyAdvisory a{id, ids_of_mask(missing), {}};
    std::string msg = "net counts for graphlet " + std::to_string(id) + " (" + kSigma16[id].name +
                      ") will include non-induced occurrences: missing supergraph(s)";
    for (int c : a.missing_supergraphs) msg += " " + std::to_string(c);
    a.message = std::move(msg);
    out.push_back(std::move(a));
  }
  return out;
}

// ===================================================================== graph
SparseAdjacency::SparseAdjacency(std::vector<std::int64_t> row_offsets,
                                 std::vector<vertex_t> col_indices)
    : offsets_(std::move(row_offsets)), cols_(std::move(col_indices)) {
  if (offsets_.empty()) offsets_.assign(1, 0);
  n_ = static_cast<vertex_t>(offsets_.size() - 1);
  m_ = static_cast<count_t>(cols_.size() / 2);
  // d_max = the largest gap between consecutive offsets
  for (std::size_t i = 1; i < offsets_.size(); ++i)
    d_max_ = std::max<vertex_t>(d_max_, offsets_[i] - offsets_[i - 1]);
}

bool SparseAdjacency::has_edge(vertex_t u, vertex_t v) const {
  const auto r = row(u);
  return std::binary_search(r.begin(), r.end(), v);
}

// The invariants of graph.hpp (zero diagonal, strictly increasing rows,
// symmetric, ids in range), reported for the first offending entry in row-
// major order with the reference's messages (proj/src/graph.cpp:173-190).
void SparseAdjacency::validate() const {
  const bool offsets_ok =
      offsets_.front() == 0 && offsets_.back() == static_cast<std::int64_t>(cols_.size());
  if (!offsets_ok) throw StructuralError("corrupt row offsets");
  auto first_problem = [this](vertex_t v) -> std::string {
    const auto r = row(v);
    for (std::size_t k = 0; k < r.size(); ++k) {
      const vertex_t x = r[k];
      if (x < 0 || x >= n_) return "column out of range";
      if (x == v) return "self-loop in adjacency";
      if (k > 0 && x <= r[k - 1]) return "row not strictly increasing";
      if (!has_edge(x, v))
        return "asymmetric adjacency at (" + std::to_string(v) + "," + std::to_string(x) + ")";
    }
    return {};
  };
  for (vertex_t v = 0; v < n_; ++v)
    if (std::string why = first_problem(v); !why.empty()) throw StructuralError(why);
}

const Csr32& SparseAdjacency::csr32() const {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (!narrow_) {
    if (n_ >= (vertex_t{1} << 31) || cols_.size() >= (std::size_t{1} << 31))
      throw StructuralError("graph exceeds the int32 CSR limits of the device path");
    auto c = std::make_shared<Csr32>();
    c->row_ptr.assign(offsets_.begin(), offsets_.end());
    c->col_idx.assign(cols_.begin(), cols_.end());
    narrow_ = std::move(c);
  }
  return *narrow_;
}

namespace {

inline bool is_blank(char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; }

// The whitespace-separated fields of one line, scanned in place: the first
// kKeep are kept, all are counted (the grammars need at most five).
struct Fields {
  static constexpr std::size_t kKeep = 8;
  std::array<std::string_view, kKeep> at{};
  std::size_t count = 0;
  explicit Fields(std::string_view line) {
    const char* p = line.data();
    const char* const e = p + line.size();
    for (;;) {
      p = std::find_if_not(p, e, is_blank);
      if (p == e) break;
      const char* q = std::find_if(p, e, is_blank);
      if (count < kKeep) at[count] = std::string_view(p, static_cast<std::size_t>(q - p));
      ++count;
      p = q;
    }
  }
  std::string_view operator[](std::size_t k) const { return at[k]; }
};

// ASCII case folding for the Matrix Market keywords.
std::string folded(std::string_view s) {
  std::string o(s.size(), '\0');
  std::transform(s.begin(), s.end(), o.begin(),
                 [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
  return o;
}

}  // namespace

// ------------------------------------------------------------ text parsers
// Same grammar, error classes and messages as the reference's serial parsers
// (proj/src/graph.cpp:52-157), parsed in parallel: the stream is read whole,
// cut into per-thread chunks at line boundaries, each chunk is parsed with
// its own first error, and the chunks are merged in file order, so the error
// reported is the one the serial parser would have thrown first.
namespace {

std::string slurp(std::istream& in) {
  std::string buf;
  constexpr std::size_t kBlock = std::size_t{1} << 24;
  for (;;) {
    const std::size_t at = buf.size();
    buf.resize(at + kBlock);
    in.read(buf.data() + at, static_cast<std::streamsize>(kBlock));
    buf.resize(at + static_cast<std::size_t>(in.gcount()));
    if (!in) break;
  }
  return buf;
}

std::string_view strip(std::string_view s) {
  const char* b = std::find_if_not(s.data(), s.data() + s.size(), is_blank);
  const char* e = s.data() + s.size();
  while (e > b && is_blank(e[-1])) --e;
  return std::string_view(b, static_cast<std::size_t>(e - b));
}

// Next line of buf starting at *pos (without the '\n'); false at the end.
bool next_line(std::string_view buf, std::size_t* pos, std::string_view* line) {
  if (*pos >= buf.size()) return false;
  const char* b = buf.data() + *pos;
  const void* nl = std::memchr(b, '\n', buf.size() - *pos);
  const std::size_t len = nl ? static_cast<std::size_t>(static_cast<const char*>(nl) - b)
                             : buf.size() - *pos;
  *line = std::string_view(b, len);
  *pos += len + (nl ? 1 : 0);
  return true;
}

struct ParsedChunk {
  std::vector<std::pair<vertex_t, vertex_t>> edges;
  std::size_t lines = 0;
  bool failed = false;
  std::size_t fail_line = 0;         // 1-based within the chunk
  std::size_t entries_before = 0;    // entries parsed before the failing line
  std::string fail_suffix;           // message after "line N"
};

// Chunks [begin, end) of buf cut at line starts.
std::vector<std::pair<std::size_t, std::size_t>> line_chunks(std::string_view buf, std::size_t from) {
  const std::size_t len = buf.size() > from ? buf.size() - from : 0;
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const std::size_t parts = std::max<std::size_t>(1, std::min<std::size_t>(hw, len >> 20));
  std::vector<std::pair<std::size_t, std::size_t>> out;
  std::size_t start = from;
  for (std::size_t k = 1; k <= parts && start < buf.size(); ++k) {
    std::size_t end = k == parts ? buf.size() : from + len * k / parts;
    if (end < start) end = start;
    if (end < buf.size()) {
      const void* nl = std::memchr(buf.data() + end, '\n', buf.size() - end);
      end = nl ? static_cast<std::size_t>(static_cast<const char*>(nl) - buf.data()) + 1 : buf.size();
    }
    out.emplace_back(start, end);
    start = end;
  }
  return out;
}

// Parse every chunk on its own thread with `entry(line_view, chunk)`.
template <class F>
std::vector<ParsedChunk> parse_chunks(std::string_view buf, std::size_t from, F entry) {
  auto cuts = line_chunks(buf, from);
  std::vector<ParsedChunk> res(cuts.size());
  auto work = [&](std::size_t k) {
    ParsedChunk& c = res[k];
    std::size_t pos = cuts[k].first;
    std::string_view whole = buf.substr(0, cuts[k].second), line;
    while (next_line(whole, &pos, &line)) {
      ++c.lines;
      if (c.failed) continue;  // keep counting lines only
      std::string suffix;
      if (!entry(strip(line), &c, &suffix)) {
        c.failed = true;
        c.fail_line = c.lines;
        c.entries_before = c.edges.size();
        c.fail_suffix = std::move(suffix);
      }
    }
  };
  std::vector<std::thread> th;
  for (std::size_t k = 1; k < cuts.size(); ++k) th.emplace_back(work, k);
  if (!cuts.empty()) work(0);
  for (auto& t : th) t.join();
  return res;
}

bool parse_i64(std::string_view t, std::int64_t* v) {
  auto r = std::from_chars(t.data(), t.data() + t.size(), *v);
  return r.ec == std::errc{} && r.ptr == t.data() + t.size();
}

}  // namespace

EdgeCollection parse_edge_list(std::istream& in) {
  const std::string buf = slurp(in);
  auto chunks = parse_chunks(buf, 0, [](std::string_view body, ParsedChunk* c, std::string* err) {
    if (body.empty() || body.front() == '#' || body.front() == '%') return true;
    const Fields t(body);
    if (t.count != 2) {
      *err = ": expected 'u v', got " + std::to_string(t.count) + " tokens";
      return false;
    }
    std::int64_t u = 0, v = 0;
    if (!parse_i64(t[0], &u)) { *err = ": malformed vertex id '" + std::string(t[0]) + "'"; return false; }
    if (!parse_i64(t[1], &v)) { *err = ": malformed vertex id '" + std::string(t[1]) + "'"; return false; }
    if (u < 0 || v < 0) { *err = ": negative vertex id"; return false; }
    c->edges.emplace_back(u, v);
    return true;
  });
  EdgeCollection ec;
  ec.origin = EdgeOrigin::kEdgeList;
  std::size_t line_base = 0, total = 0;
  for (auto& c : chunks) {
    if (c.failed) throw ParseError("line " + std::to_string(line_base + c.fail_line) + c.fail_suffix);
    line_base += c.lines;
    total += c.edges.size();
  }
  ec.edges.reserve(total);
  for (auto& c : chunks) ec.edges.insert(ec.edges.end(), c.edges.begin(), c.edges.end());
  return ec;
}

EdgeCollection parse_matrix_market(std::istream& in) {
  const std::string buf = slurp(in);
  std::size_t pos = 0, ln = 0;
  std::string_view line;
  if (!next_line(buf, &pos, &line)) throw ParseError("empty Matrix Market stream");
  ++ln;
  const Fields banner(line);
  if (banner.count < 5 || folded(banner[0]) != "%%matrixmarket" || folded(banner[1]) != "matrix")
    throw ParseError("line 1: missing %%MatrixMarket matrix banner");
  const std::string format = folded(banner[2]), field = folded(banner[3]), sym = folded(banner[4]);
  if (format != "coordinate")
    throw ParseError("line 1: only coordinate format is supported, got '" + format + "'");
  if (field != "pattern" && field != "real" && field != "integer")
    throw ParseError("line 1: unsupported field '" + field + "'");
  if (sym != "general" && sym != "symmetric")
    throw ParseError("line 1: unsupported symmetry '" + sym + "'");
  const std::size_t per_entry = field == "pattern" ? 2 : 3;
  // size line, after any comments (only '%' lines are comments here)
  std::int64_t rows = 0, cols = 0, nnz = 0;
  for (;;) {
    if (!next_line(buf, &pos, &line)) throw ParseError("unexpected end of stream before size line");
    ++ln;
    const std::string_view body = strip(line);
    if (body.empty() || body.front() == '%') continue;
    const Fields t(body);
    if (t.count != 3) throw ParseError("line " + std::to_string(ln) + ": expected 'rows cols nnz'");
    const char* const what[3] = {"row count", "column count", "entry count"};
    std::int64_t* const dst[3] = {&rows, &cols, &nnz};
    for (int k = 0; k < 3; ++k)
      if (!parse_i64(t[k], dst[k]))
        throw ParseError("line " + std::to_string(ln) + ": malformed " + what[k] + " '" +
                         std::string(t[k]) + "'");
    break;
  }
  if (rows != cols)
    throw ParseError("dimension mismatch: adjacency must be square, got " + std::to_string(rows) +
                     "x" + std::to_string(cols));
  if (rows < 0 || nnz < 0) throw ParseError("negative size header");
  auto chunks = parse_chunks(buf, pos, [&](std::string_view body, ParsedChunk* c, std::string* err) {
    if (body.empty() || body.front() == '%') return true;
    const Fields t(body);
    if (t.count != per_entry) {
      *err = ": expected " + std::to_string(per_entry) + " tokens per entry";
      return false;
    }
    std::int64_t i = 0, j = 0;
    if (!parse_i64(t[0], &i)) { *err = ": malformed row index '" + std::string(t[0]) + "'"; return false; }
    if (!parse_i64(t[1], &j)) { *err = ": malformed column index '" + std::string(t[1]) + "'"; return false; }
    if (i < 1 || i > rows || j < 1 || j > cols) {
      *err = ": entry (" + std::to_string(i) + "," + std::to_string(j) + ") out of declared range " +
             std::to_string(rows);
      return false;
    }
    c->edges.emplace_back(i - 1, j - 1);
    return true;
  });
  EdgeCollection ec;
  ec.origin = sym == "symmetric" ? EdgeOrigin::kMatrixMarketSymmetric : EdgeOrigin::kMatrixMarketGeneral;
  ec.declared_n = rows;
  // the serial parser stops after nnz entries: later lines (even malformed ones) are never read
  std::int64_t seen = 0;
  std::size_t line_base = ln;
  for (auto& c : chunks) {
    if (seen >= nnz) break;
    if (c.failed && seen + static_cast<std::int64_t>(c.entries_before) < nnz)
      throw ParseError("line " + std::to_string(line_base + c.fail_line) + c.fail_suffix);
    const std::int64_t take = std::min<std::int64_t>(static_cast<std::int64_t>(c.edges.size()), nnz - seen);
    ec.edges.insert(ec.edges.end(), c.edges.begin(), c.edges.begin() + take);
    seen += take;
    line_base += c.lines;
  }
  if (seen < nnz)
    throw ParseError("unexpected end of stream: got " + std::to_string(seen) + " of " +
                     std::to_string(nnz) + " entries");
  return ec;
}

namespace {
BuildResult device_ingest(const EdgeCollection& ec, const SanitizeOptions& opt);
}  // namespace

// Sanitised CSR from an edge collection: mirror, drop self-loops, sort,
// dedupe, offsets — all on the device (fglt_build_csr, fglt_ingest.cuh), with
// build_adjacency's error classes, messages and BuildReport
// (proj/src/graph.cpp:192-249). There is no host path: without a CUDA device
// this throws, like every other entry point.
BuildResult build_adjacency(const EdgeCollection& ec, const SanitizeOptions& opt) {
  return device_ingest(ec, opt);
}

std::vector<count_t> degree_vector(const SparseAdjacency& g) {
  std::vector<count_t> d(static_cast<std::size_t>(g.num_vertices()));
  for (vertex_t v = 0; v < g.num_vertices(); ++v) d[v] = static_cast<count_t>(g.degree(v));
  return d;
}

// ================================================================ conversion
// A conversion matrix is checked once (unit diagonal, nothing below it, in
// row-major order) and keeps, per row, its nonzero entries right of the
// diagonal: the only ones back substitution and apply_conversion read.
ConversionMatrix::ConversionMatrix(std::vector<int> ids, std::vector<std::vector<count_t>> dense)
    : ids_(std::move(ids)), dense_(std::move(dense)), tails_(ids_.size()) {
  const std::size_t k = ids_.size();
  for (std::size_t r = 0; r < k; ++r) {
    const auto& row = dense_[r];
    if (row[r] != 1) throw Error("conversion matrix is not unit-diagonal at row " + std::to_string(r));
    const auto below = std::find_if(row.begin(), row.begin() + static_cast<std::ptrdiff_t>(r),
                                    [](count_t x) { return x != 0; });
    if (below != row.begin() + static_cast<std::ptrdiff_t>(r))
      throw Error("conversion matrix is not upper triangular at (" + std::to_string(r) + "," +
                  std::to_string(below - row.begin()) + ")");
    for (std::size_t c = r + 1; c < k; ++c)
      if (row[c]) tails_[r].emplace_back(c, row[c]);
  }
}

ConversionMatrix sub_matrix(const Dictionary& d) {
  const auto& ids = d.ids();
  std::vector<std::vector<count_t>> m(ids.size());
  for (std::size_t r = 0; r < ids.size(); ++r)
    for (int c : ids) m[r].push_back(fglt_tables::u16_coef(ids[r], c));
  return ConversionMatrix(ids, std::move(m));
}

const ConversionMatrix& full_u16() {
  static const ConversionMatrix u = sub_matrix(Dictionary::all());
  return u;
}

RawFrequencyField apply_conversion(const NetFrequencyField& net, const ConversionMatrix& U) {
  if (net.dictionary().ids() != U.ids())
    throw Error("conversion matrix does not match the field's dictionary");
  RawFrequencyField raw(net.num_vertices(), net.dictionary());
  for (vertex_t v = 0; v < net.num_vertices(); ++v) {
    auto in = net.vertex_row(v);
    auto out = raw.vertex_row(v);
    for (std::size_t r = 0; r < U.dim(); ++r) {
      count_t acc = in[r];
      for (auto [c, k] : U.row_tail(r))
        acc = checked_add(acc, checked_mul(k, in[c], U.ids()[r], v), U.ids()[r], v);
      out[r] = acc;
    }
  }
  return raw;
}

bool inverse_pattern_check(const ConversionMatrix& U) {
  const std::size_t k = U.dim();
  // exact integer inverse, column by column (unit upper triangular)
  std::vector<std::vector<std::int64_t>> inv(k, std::vector<std::int64_t>(k, 0));
  for (std::size_t col = 0; col < k; ++col)
    for (std::size_t r = k; r-- > 0;) {
      std::int64_t x = r == col ? 1 : 0;
      for (auto [c, coef] : U.row_tail(r)) x -= static_cast<std::int64_t>(coef) * inv[c][col];
      inv[r][col] = x;
    }
  for (std::size_t r = 0; r < k; ++r)
    for (std::size_t c = 0; c < k; ++c)
      if (inv[r][c] && !U.coeff(r, c)) return false;  // fill-in outside U's pattern
  for (std::size_t r = 0; r < k; ++r)
    for (std::size_t j = r + 1; j < k; ++j)
      if (U.coeff(r, j))
        for (std::size_t c = j + 1; c < k; ++c)
          if (U.coeff(j, c) && !U.coeff(r, c)) return false;  // not transitively closed
  return true;
}

// ============================================================ device bridge
namespace {

std::mutex g_ctx_mu;
std::map<int, fglt_ctx*> g_ctx;
std::mutex g_run_mu;  // one device call per context at a time

fglt_ctx* context_for(int device) {
  std::lock_guard<std::mutex> lock(g_ctx_mu);
  auto it = g_ctx.find(device);
  if (it != g_ctx.end()) return it->second;
  fglt_error err{};
  fglt_ctx* c = fglt_ctx_create(device, nullptr, &err);
  if (!c) throw Error(std::string("CUDA device unavailable: ") + err.msg);
  g_ctx[device] = c;
  return c;
}

[[noreturn]] void rethrow(int rc, const fglt_error& e);

BuildResult device_ingest(const EdgeCollection& ec, const SanitizeOptions& opt) {
  fglt_ctx* ctx = context_for(0);
  const std::size_t ne = ec.edges.size();
  std::vector<std::int64_t> eu(ne), ev(ne);
  for (std::size_t i = 0; i < ne; ++i) {
    eu[i] = ec.edges[i].first;
    ev[i] = ec.edges[i].second;
  }
  std::int64_t n = 0, nnz = 0, loops = 0, dups = 0;
  fglt_error err{};
  std::vector<std::int32_t> rp, ci;
  {
    std::lock_guard<std::mutex> lock(g_run_mu);
    int rc = fglt_build_csr(ctx, eu.data(), ev.data(), static_cast<std::int64_t>(ne),
                            ec.declared_n.value_or(0), opt.symmetrize || ec.declared_symmetric(),
                            opt.drop_self_loops, opt.dedupe, 0, &n, &nnz, &loops, &dups, &err);
    if (rc) rethrow(rc, err);
    rp.resize(static_cast<std::size_t>(n) + 1);
    ci.resize(static_cast<std::size_t>(nnz));
    rc = fglt_csr_fetch(ctx, rp.data(), ci.data(), 0, &err);
    if (rc) rethrow(rc, err);
  }
  BuildResult out;
  out.graph = SparseAdjacency(std::vector<std::int64_t>(rp.begin(), rp.end()),
                              std::vector<vertex_t>(ci.begin(), ci.end()));
  out.report.self_loops_dropped = static_cast<count_t>(loops);
  out.report.duplicates_merged = static_cast<count_t>(dups);
  return out;
}

[[noreturn]] void rethrow(int rc, const fglt_error& e) {
  switch (rc) {
    case FGLT_E_PARSE: throw ParseError(e.msg);
    case FGLT_E_STRUCTURAL: throw StructuralError(e.msg);
    case FGLT_E_OVERFLOW: throw OverflowError(e.msg, e.graphlet_id, e.vertex);
    case FGLT_E_INCONSISTENCY: throw InconsistencyError(e.msg, e.graphlet_id, e.vertex);
    case FGLT_E_IO: throw IoError(e.msg);
    default: throw Error(std::string("device transform failed: ") + e.msg);
  }
}

TransformStats stats_of(const fglt_stats& s) {
  TransformStats t;
  for (int i = 0; i < s.num_steps; ++i) t.kernel_times.push_back({s.step_names[i], s.step_seconds[i]});
  t.p2_row_touches = s.p2_row_touches;
  t.p2_touch_bound = s.p2_touch_bound;
  t.peak_aux_words = s.peak_aux_words;
  t.largest_aux_alloc_words = s.largest_aux_alloc_words;
  t.threads_used = s.threads_used;
  return t;
}


void run(const SparseAdjacency& g, const Dictionary& dict, bool lenient, int device,
         count_t* raw, count_t* net, TransformStats* stats) {
  const Csr32& c = g.csr32();
  fglt_ctx* ctx = context_for(device);
  fglt_stats st{};
  fglt_error err{};
  int rc;
  {
    std::lock_guard<std::mutex> lock(g_run_mu);
    rc = fglt_ctx_transform(ctx, c.row_ptr.data(), c.col_idx.data(), g.num_vertices(),
                            static_cast<std::int64_t>(c.col_idx.size()), dict.mask(), lenient ? 1 : 0,
                            stats ? FGLT_TIMINGS : 0u, raw, net, stats ? &st : nullptr, &err);
  }
  if (rc) rethrow(rc, err);
  if (stats) *stats = stats_of(st);
}

}  // namespace

RawFrequencyField raw_frequencies(const SparseAdjacency& g, const Dictionary& dict,
                                  const KernelOptions& opt, TransformStats* stats) {
  RawFrequencyField raw(g.num_vertices(), dict);
  TransformStats st;
  // lenient: raw columns must not depend on whether the family is complete
  run(g, dict, /*lenient=*/true, opt.device, raw.mutable_data(), nullptr, &st);
  // the conversion step is not part of raw_frequencies
  if (!st.kernel_times.empty() && st.kernel_times.back().name == "conversion")
    st.kernel_times.pop_back();
  if (stats) *stats = st;
  return raw;
}

TransformResult transform(const SparseAdjacency& g, const TransformOptions& opt) {
  TransformResult r{RawFrequencyField(g.num_vertices(), opt.dict),
                    NetFrequencyField(g.num_vertices(), opt.dict), {}};
  if (opt.devices.size() > 1) {  // single-process multi-GPU (fglt_multi.cpp)
    const Csr32& c = g.csr32();
    fglt_stats st{};
    fglt_error err{};
    const int rc = fglt_transform_multi(
        c.row_ptr.data(), c.col_idx.data(), g.num_vertices(),
        static_cast<std::int64_t>(c.col_idx.size()), opt.dict.mask(), opt.lenient ? 1 : 0,
        opt.devices.data(), static_cast<int>(opt.devices.size()), 0u, r.raw.mutable_data(),
        r.net.mutable_data(), &st, &err);
    if (rc) rethrow(rc, err);
    r.stats = stats_of(st);
    return r;
  }
  run(g, opt.dict, opt.lenient, opt.device, r.raw.mutable_data(), r.net.mutable_data(), &r.stats);
  return r;
}

void release_device_workspace() {
  std::lock_guard<std::mutex> lock(g_ctx_mu);
  std::lock_guard<std::mutex> run(g_run_mu);
  for (auto& kv : g_ctx) fglt_ctx_release_workspace(kv.second);
}

NetFrequencyField net_from_raw(const RawFrequencyField& raw, const ConversionMatrix& U,
                               bool lenient, int /*threads*/) {
  if (raw.dictionary().ids() != U.ids())
    throw Error("conversion matrix does not match the field's dictionary");
  NetFrequencyField net(raw.num_vertices(), raw.dictionary());
  if (raw.num_vertices() == 0) return net;
  // the matrix the caller passed, not the built-in U16(s,s) (conversion.cpp:80-116)
  const std::size_t k = U.dim();
  std::vector<count_t> dense(k * k);
  for (std::size_t r = 0; r < k; ++r)
    for (std::size_t c = 0; c < k; ++c) dense[r * k + c] = U.coeff(r, c);
  fglt_ctx* ctx = context_for(0);
  fglt_error err{};
  int rc;
  {
    std::lock_guard<std::mutex> lock(g_run_mu);
    rc = fglt_net_from_raw_matrix(ctx, raw.data().data(), raw.num_vertices(),
                                  raw.dictionary().mask(), dense.data(), lenient ? 1 : 0,
                                  net.mutable_data(), &err);
  }
  if (rc) rethrow(rc, err);
  return net;
}

// ============================================================ per-kernel API
// The reference's public per-kernel functions (kernels.hpp:43-98), each one
// device call through the C-ABI (fglt_kernel_*, fglt_kernels_api.cuh) or a
// column of the device transform. `threads` is accepted for source
// compatibility only.
namespace {

template <class F>
void device_call(F&& f) {
  fglt_ctx* ctx = context_for(0);
  fglt_error err{};
  int rc;
  {
    std::lock_guard<std::mutex> lock(g_run_mu);
    rc = f(ctx, &err);
  }
  if (rc) rethrow(rc, err);
}

void need_size(const std::vector<count_t>& v, vertex_t n, const char* what) {
  if (static_cast<vertex_t>(v.size()) < n)
    throw Error(std::string(what) + " is shorter than the vertex count");
}

std::vector<count_t> column(const RawFrequencyField& f, int id) {
  std::vector<count_t> out(static_cast<std::size_t>(f.num_vertices()));
  const std::size_t c = f.dictionary().position_of(id);
  for (vertex_t v = 0; v < f.num_vertices(); ++v) out[v] = f.at(v, c);
  return out;
}

}  // namespace

std::vector<count_t> compute_p2(const SparseAdjacency& g, const std::vector<count_t>& p1, int) {
  const vertex_t n = g.num_vertices();
  need_size(p1, n, "p1");
  std::vector<count_t> p2(static_cast<std::size_t>(n));
  const Csr32& c = g.csr32();
  device_call([&](fglt_ctx* ctx, fglt_error* e) {
    return fglt_kernel_p2(ctx, c.row_ptr.data(), c.col_idx.data(), n,
                          static_cast<std::int64_t>(c.col_idx.size()), p1.data(), p2.data(), e);
  });
  return p2;
}

std::pair<std::vector<count_t>, SparseCountMatrix> compute_c3_C3(const SparseAdjacency& g, int) {
  const vertex_t n = g.num_vertices();
  const Csr32& c = g.csr32();
  std::vector<count_t> c3(static_cast<std::size_t>(n)), C3(c.col_idx.size());
  device_call([&](fglt_ctx* ctx, fglt_error* e) {
    return fglt_kernel_c3(ctx, c.row_ptr.data(), c.col_idx.data(), n,
                          static_cast<std::int64_t>(c.col_idx.size()), c3.data(), C3.data(), e);
  });
  return {std::move(c3), SparseCountMatrix(g, std::move(C3))};
}

std::vector<count_t> compute_p3(const SparseAdjacency& g, const std::vector<count_t>& p1,
                                const std::vector<count_t>& p2, const std::vector<count_t>& c3,
                                int) {
  const vertex_t n = g.num_vertices();
  need_size(p1, n, "p1");
  need_size(p2, n, "p2");
  need_size(c3, n, "c3");
  std::vector<count_t> p3(static_cast<std::size_t>(n));
  const Csr32& c = g.csr32();
  device_call([&](fglt_ctx* ctx, fglt_error* e) {
    return fglt_kernel_p3(ctx, c.row_ptr.data(), c.col_idx.data(), n,
                          static_cast<std::int64_t>(c.col_idx.size()), p1.data(), p2.data(),
                          c3.data(), p3.data(), e);
  });
  return p3;
}

FourCycleResult compute_c4_d14(const SparseAdjacency& g, int) {
  const int ids[] = {12, 14};
  TransformStats st;
  RawFrequencyField raw = raw_frequencies(g, Dictionary::from_ids(ids), {}, &st);
  FourCycleResult r;
  r.c4 = column(raw, 12);
  r.d14 = column(raw, 14);
  r.accumulator_touches = st.p2_row_touches;
  return r;
}

std::vector<count_t> compute_d7(const SparseAdjacency& g, const std::vector<count_t>& p1, int) {
  const vertex_t n = g.num_vertices();
  need_size(p1, n, "p1");
  std::vector<count_t> d7(static_cast<std::size_t>(n));
  const Csr32& c = g.csr32();
  device_call([&](fglt_ctx* ctx, fglt_error* e) {
    return fglt_kernel_d7(ctx, c.row_ptr.data(), c.col_idx.data(), n,
                          static_cast<std::int64_t>(c.col_idx.size()), p1.data(), d7.data(), e);
  });
  return d7;
}

std::vector<count_t> compute_d8(const std::vector<count_t>& p1, int) {
  std::vector<count_t> d8(p1.size());
  if (p1.empty()) return d8;
  device_call([&](fglt_ctx* ctx, fglt_error* e) {
    return fglt_kernel_d8(ctx, static_cast<std::int64_t>(p1.size()), p1.data(), d8.data(), e);
  });
  return d8;
}

DipperCounts compute_d9_d10_d11(const SparseAdjacency& g, const std::vector<count_t>& p1,
                                const std::vector<count_t>& c3, const SparseCountMatrix& C3,
                                int) {
  const vertex_t n = g.num_vertices();
  need_size(p1, n, "p1");
  need_size(c3, n, "c3");
  const Csr32& c = g.csr32();
  if (C3.values().size() != c.col_idx.size())
    throw Error("C3 does not share the graph's CSR pattern");
  DipperCounts r;
  r.d9.resize(static_cast<std::size_t>(n));
  r.d10.resize(static_cast<std::size_t>(n));
  r.d11.resize(static_cast<std::size_t>(n));
  device_call([&](fglt_ctx* ctx, fglt_error* e) {
    return fglt_kernel_d9_d10_d11(ctx, c.row_ptr.data(), c.col_idx.data(), n,
                                  static_cast<std::int64_t>(c.col_idx.size()), p1.data(),
                                  c3.data(), C3.values().data(), r.d9.data(), r.d10.data(),
                                  r.d11.data(), e);
  });
  return r;
}

std::vector<count_t> compute_d13(const SparseAdjacency& g, const SparseCountMatrix& C3, int) {
  const vertex_t n = g.num_vertices();
  const Csr32& c = g.csr32();
  if (C3.values().size() != c.col_idx.size())
    throw Error("C3 does not share the graph's CSR pattern");
  std::vector<count_t> d13(static_cast<std::size_t>(n));
  device_call([&](fglt_ctx* ctx, fglt_error* e) {
    return fglt_kernel_d13(ctx, c.row_ptr.data(), c.col_idx.data(), n,
                           static_cast<std::int64_t>(c.col_idx.size()), C3.values().data(),
                           d13.data(), e);
  });
  return d13;
}

std::vector<count_t> compute_d15(const SparseAdjacency& g, int) {
  const int ids[] = {15};
  return column(raw_frequencies(g, Dictionary::from_ids(ids)), 15);
}

}  // namespace graphlet
