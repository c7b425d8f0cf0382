// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin C-ABI over the UNMODIFIED reference library, compiled by
// oracle/Makefile from the sources where they lie under
// /root/reference/proj/src (nothing is copied into this repo). Output goes to
// oracle/_ref/libfglt_ref.so, which is git-ignored but travels to the GPU box.
//
// Used as (1) the pin for the oracle restatement (oracle/fglt_oracle.c) and
// the golden fixtures, and (2) the CPU baseline / `bench.py --impl reference`
// arm. Each entry point wraps exactly one reference call:
//   fglt_ref_transform_csr32  -> graphlet::transform     (proj/src/transform.cpp:9-26)
//   fglt_ref_er_graph          -> testutil::er_graph      (proj/tests/testutil.hpp:90-99)
//   fglt_ref_oracle_raw/net    -> graphlet::oracle_raw/net (proj/src/oracle.cpp:102-308)
//   fglt_ref_build_adjacency   -> graphlet::build_adjacency (proj/src/graph.cpp:192-249)
//   fglt_ref_count_*           -> whole-graph tallies     (proj/src/oracle.cpp:359-407)
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "graphlet/oracle.hpp"
#include "graphlet/transform.hpp"
#include "testutil.hpp"

using namespace graphlet;

namespace {

std::string g_last_stats;

SparseAdjacency wrap(const int32_t* rp, const int32_t* ci, int64_t n,
                     int64_t nnz) {
  std::vector<std::int64_t> off(rp, rp + n + 1);
  std::vector<vertex_t> col(ci, ci + nnz);
  return SparseAdjacency(std::move(off), std::move(col));
}

Dictionary dict_of(uint32_t mask) {
  std::vector<int> ids;
  for (int i = 0; i < kNumGraphlets; ++i)
    if (mask & (1u << i)) ids.push_back(i);
  return Dictionary::from_ids(std::span<const int>(ids.data(), ids.size()));
}

void put_msg(char* msg, int len, const std::string& s) {
  if (!msg || len <= 0) return;
  std::strncpy(msg, s.c_str(), static_cast<std::size_t>(len - 1));
  msg[len - 1] = 0;
}

}  // namespace

extern "C" {

// Return codes follow the reference CLI's exit classes (tools/glt.cpp:17-21):
// 0 ok, 1 parse, 2 structural, 3 overflow, 4 inconsistency, 6 other.
int fglt_ref_transform_csr32(const int32_t* rp, const int32_t* ci, int64_t n,
                             int64_t nnz, uint32_t dict_mask, int lenient,
                             int threads, uint64_t* raw_out, uint64_t* net_out,
                             double* seconds, int32_t* err_graphlet,
                             int64_t* err_vertex, char* msg, int msglen) {
  try {
    SparseAdjacency g = wrap(rp, ci, n, nnz);
    TransformOptions opt;
    opt.dict = dict_of(dict_mask);
    opt.threads = threads;
    opt.lenient = lenient != 0;
    auto t0 = std::chrono::steady_clock::now();
    TransformResult r = transform(g, opt);
    auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (raw_out)
      std::memcpy(raw_out, r.raw.data().data(),
                  r.raw.data().size() * sizeof(uint64_t));
    if (net_out)
      std::memcpy(net_out, r.net.data().data(),
                  r.net.data().size() * sizeof(uint64_t));
    std::ostringstream js;
    js << "{\"threads_used\": " << r.stats.threads_used
       << ", \"p2_row_touches\": " << r.stats.p2_row_touches
       << ", \"p2_touch_bound\": " << r.stats.p2_touch_bound
       << ", \"peak_aux_words\": " << r.stats.peak_aux_words
       << ", \"largest_aux_alloc_words\": " << r.stats.largest_aux_alloc_words
       << ", \"kernel_times\": [";
    for (std::size_t i = 0; i < r.stats.kernel_times.size(); ++i)
      js << (i ? ", " : "") << "[\"" << r.stats.kernel_times[i].name << "\", "
         << r.stats.kernel_times[i].seconds << "]";
    js << "]}";
    g_last_stats = js.str();
    return 0;
  } catch (const ParseError& e) {
    put_msg(msg, msglen, e.what());
    return 1;
  } catch (const StructuralError& e) {
    put_msg(msg, msglen, e.what());
    return 2;
  } catch (const OverflowError& e) {
    if (err_graphlet) *err_graphlet = e.graphlet_id;
    if (err_vertex) *err_vertex = e.vertex;
    put_msg(msg, msglen, e.what());
    return 3;
  } catch (const InconsistencyError& e) {
    if (err_graphlet) *err_graphlet = e.graphlet_id;
    if (err_vertex) *err_vertex = e.vertex;
    put_msg(msg, msglen, e.what());
    return 4;
  } catch (const std::exception& e) {
    put_msg(msg, msglen, e.what());
    return 6;
  }
}

const char* fglt_ref_last_stats(void) { return g_last_stats.c_str(); }

// parse_dictionary (proj/src/dictionary.cpp): ids and implicitly added ids
// as bit masks; returns 0 or 1 (ParseError, message in msg).
int fglt_ref_parse_dictionary(const char* spec, uint32_t* ids_mask, uint32_t* implicit_mask,
                              char* msg, int msglen) {
  try {
    ParsedDictionary p = parse_dictionary(spec);
    *ids_mask = 0;
    for (int id : p.dict.ids()) *ids_mask |= 1u << id;
    *implicit_mask = 0;
    for (int id : p.implicitly_added) *implicit_mask |= 1u << id;
    return 0;
  } catch (const ParseError& e) {
    put_msg(msg, msglen, e.what());
    return 1;
  }
}

// build_adjacency (proj/src/graph.cpp:192-249) on (eu[i], ev[i]) pairs with
// SanitizeOptions; rp/ci caller-allocated (n_max + 1, 2 ne); out4 = {n, nnz,
// self_loops_dropped, duplicates_merged}. Returns 0 or 2 (StructuralError).
int fglt_ref_build_adjacency(const int64_t* eu, const int64_t* ev, int64_t ne,
                             int64_t declared_n, int symmetrize, int drop_self_loops,
                             int dedupe, int32_t* rp, int32_t* ci, int64_t* out4,
                             char* msg, int msglen) {
  try {
    EdgeCollection ec;
    ec.edges.reserve(static_cast<std::size_t>(ne));
    for (int64_t i = 0; i < ne; ++i) ec.edges.emplace_back(eu[i], ev[i]);
    if (declared_n > 0) ec.declared_n = declared_n;
    SanitizeOptions o;
    o.symmetrize = symmetrize != 0;
    o.drop_self_loops = drop_self_loops != 0;
    o.dedupe = dedupe != 0;
    BuildResult b = build_adjacency(ec, o);
    const auto& off = b.graph.row_offsets();
    const auto& col = b.graph.col_indices();
    for (std::size_t i = 0; i < off.size(); ++i) rp[i] = static_cast<int32_t>(off[i]);
    for (std::size_t i = 0; i < col.size(); ++i) ci[i] = static_cast<int32_t>(col[i]);
    out4[0] = b.graph.num_vertices();
    out4[1] = static_cast<int64_t>(col.size());
    out4[2] = static_cast<int64_t>(b.report.self_loops_dropped);
    out4[3] = static_cast<int64_t>(b.report.duplicates_merged);
    return 0;
  } catch (const StructuralError& e) {
    put_msg(msg, msglen, e.what());
    return 2;
  } catch (const std::exception& e) {
    put_msg(msg, msglen, e.what());
    return 6;
  }
}

// er_graph(n, p, seed): first call with rp == nullptr to learn nnz.
int64_t fglt_ref_er_graph(int64_t n, double p, uint64_t seed, int32_t* rp,
                          int32_t* ci) {
  SparseAdjacency g = testutil::er_graph(n, p, seed);
  const auto& off = g.row_offsets();
  const auto& col = g.col_indices();
  if (rp) {
    for (std::size_t i = 0; i < off.size(); ++i) rp[i] = static_cast<int32_t>(off[i]);
    for (std::size_t i = 0; i < col.size(); ++i) ci[i] = static_cast<int32_t>(col[i]);
  }
  return static_cast<int64_t>(col.size());
}

// Brute-force oracles (n <= 200), full 16 columns.
int fglt_ref_oracle(const int32_t* rp, const int32_t* ci, int64_t n,
                    int64_t nnz, uint64_t* raw_out, uint64_t* net_out) {
  try {
    SparseAdjacency g = wrap(rp, ci, n, nnz);
    if (raw_out) {
      auto r = oracle_raw(g);
      std::memcpy(raw_out, r.data().data(), r.data().size() * 8);
    }
    if (net_out) {
      auto r = oracle_net(g);
      std::memcpy(net_out, r.data().data(), r.data().size() * 8);
    }
    return 0;
  } catch (const std::exception&) {
    return 2;
  }
}

void fglt_ref_counts(const int32_t* rp, const int32_t* ci, int64_t n,
                     int64_t nnz, uint64_t* out3) {
  SparseAdjacency g = wrap(rp, ci, n, nnz);
  out3[0] = count_triangles(g);
  out3[1] = count_four_cycles(g);
  out3[2] = count_tetrahedra(g);
}

// The reference's own d15 kernel alone (proj/src/kernels.cpp:234-288), used
// to pin the independent K4 counter at scales where the full transform is
// out of reach.
int fglt_ref_d15(const int32_t* rp, const int32_t* ci, int64_t n, int64_t nnz,
                 int threads, uint64_t* out) {
  SparseAdjacency g = wrap(rp, ci, n, nnz);
  auto d = compute_d15(g, threads);
  std::memcpy(out, d.data(), d.size() * 8);
  return 0;
}

}  // extern "C"
