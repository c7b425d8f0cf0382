// brute.cpp — host brute-force graphlet oracle (include/graphlet/oracle.hpp),
// the debugging aid the reference exposes as oracle_raw / oracle_net /
// cross_check (proj/include/graphlet/oracle.hpp, bindings/module.cpp:155-179).
// It never runs on the transform path and shares no code with the device
// kernels.
//
// Method (independent of the reference's canonical-code tables):
//  * every connected vertex set S with |S| <= 4 is visited exactly once by
//    ESU enumeration (extend a set from its smallest vertex v through the
//    exclusive neighbourhoods of the members, ids > v);
//  * net: S with its induced edges is one induced graphlet; each member is
//    classified by (|S|, #edges, its degree in S, cycle/star shape);
//  * raw: every edge subset of G[S] that is connected and spans S is one
//    graphlet copy (subgraph embedding); each member is classified the same
//    way. So raw counts copies, net counts induced copies, and U·net = raw is
//    a genuine third check (cross_check leg 3).
#include <algorithm>
#include <array>
#include <sstream>
#include <vector>

#include "graphlet/conversion.hpp"
#include "graphlet/oracle.hpp"

namespace graphlet {
namespace {

// the 6 vertex pairs of a local set of <= 4 members
constexpr int kPairA[6] = {0, 0, 0, 1, 1, 2};
constexpr int kPairB[6] = {1, 2, 3, 2, 3, 3};

// Orbit of member `who` in the connected graphlet on k local vertices with
// pair mask `em` (bits over kPair*).
int orbit_of(int k, unsigned em, int who) {
  int deg[4] = {0, 0, 0, 0}, e = 0;
  for (int p = 0; p < 6; ++p)
    if (em >> p & 1u) {
      ++deg[kPairA[p]];
      ++deg[kPairB[p]];
      ++e;
    }
  const int d = deg[who];
  if (k == 1) return 0;
  if (k == 2) return 1;
  if (k == 3) return e == 3 ? 4 : (d == 1 ? 2 : 3);
  int dmax = 0, d2 = 0;
  for (int i = 0; i < 4; ++i) {
    dmax = std::max(dmax, deg[i]);
    d2 += deg[i] == 2;
  }
  switch (e) {
    case 3: return dmax == 3 ? (d == 3 ? 8 : 7) : (d == 1 ? 5 : 6);  // star / path
    case 4: return d2 == 4 ? 12 : (d == 1 ? 9 : d == 2 ? 10 : 11);   // cycle / tailed triangle
    case 5: return d == 2 ? 13 : 14;                                   // diamond
    default: return 15;                                                // clique
  }
}

bool spans_connected(int k, unsigned em) {
  unsigned reach = 1u, grow = 1u;
  while (grow) {
    unsigned next = 0;
    for (int p = 0; p < 6; ++p)
      if (em >> p & 1u) {
        const unsigned a = 1u << kPairA[p], b = 1u << kPairB[p];
        if ((grow & a) && !(reach & b)) next |= b;
        if ((grow & b) && !(reach & a)) next |= a;
      }
    reach |= next;
    grow = next;
  }
  return reach == (1u << k) - 1u;
}

// Connected sets of <= 4 vertices, each once, with their induced pair masks.
template <class F>
void for_each_connected_set(const SparseAdjacency& g, F&& visit) {
  const vertex_t n = g.num_vertices();
  std::array<vertex_t, 4> sub{};
  auto induced = [&](int k) {
    unsigned em = 0;
    for (int p = 0; p < 6; ++p)
      if (kPairB[p] < k && g.has_edge(sub[kPairA[p]], sub[kPairB[p]])) em |= 1u << p;
    return em;
  };
  auto in_or_next_to = [&](vertex_t u, int k) {
    for (int i = 0; i < k; ++i)
      if (sub[i] == u || g.has_edge(sub[i], u)) return true;
    return false;
  };
  // ESU: extend the set sub[0..k) by each candidate of ext (all > root)
  auto extend = [&](auto&& self, int k, std::vector<vertex_t> ext, vertex_t root) -> void {
    visit(sub, k, induced(k));
    if (k == 4) return;
    while (!ext.empty()) {
      const vertex_t w = ext.back();
      ext.pop_back();
      std::vector<vertex_t> next = ext;
      for (vertex_t u : g.row(w))
        if (u > root && !in_or_next_to(u, k)) next.push_back(u);
      sub[k] = w;
      self(self, k + 1, std::move(next), root);
    }
  };
  for (vertex_t v = 0; v < n; ++v) {
    sub[0] = v;
    std::vector<vertex_t> ext;
    for (vertex_t u : g.row(v))
      if (u > v) ext.push_back(u);
    extend(extend, 1, std::move(ext), v);
  }
}

void check_cap(const SparseAdjacency& g, const OracleOptions& opt) {
  if (g.num_vertices() > opt.cap)
    throw StructuralError("oracle cap exceeded: " + std::to_string(g.num_vertices()) +
                          " vertices > " + std::to_string(opt.cap));
}

}  // namespace

NetFrequencyField oracle_net(const SparseAdjacency& g, OracleOptions opt) {
  check_cap(g, opt);
  NetFrequencyField f(g.num_vertices(), Dictionary::all());
  for_each_connected_set(g, [&](const std::array<vertex_t, 4>& s, int k, unsigned em) {
    for (int i = 0; i < k; ++i) ++f.at(s[i], static_cast<std::size_t>(orbit_of(k, em, i)));
  });
  return f;
}

RawFrequencyField oracle_raw(const SparseAdjacency& g, OracleOptions opt) {
  check_cap(g, opt);
  RawFrequencyField f(g.num_vertices(), Dictionary::all());
  for_each_connected_set(g, [&](const std::array<vertex_t, 4>& s, int k, unsigned em) {
    // every sub-mask of the induced edges that is a connected spanning graph
    for (unsigned sub = em;; sub = (sub - 1) & em) {
      if (__builtin_popcount(sub) >= k - 1 && spans_connected(k, sub))
        for (int i = 0; i < k; ++i) ++f.at(s[i], static_cast<std::size_t>(orbit_of(k, sub, i)));
      if (sub == 0) break;
    }
  });
  return f;
}

std::string CrossCheckReport::summary() const {
  std::ostringstream out;
  out << "leg 1 (fast raw == oracle raw):  " << (raw_ok ? "pass" : "FAIL") << "\n";
  out << "leg 2 (fast net == oracle net):  " << (net_ok ? "pass" : "FAIL") << "\n";
  out << "leg 3 (U * oracle net == oracle raw): " << (conversion_ok ? "pass" : "FAIL") << "\n";
  if (first_mismatch)
    out << "first mismatch [" << first_mismatch->leg << "] vertex " << first_mismatch->vertex
        << ", graphlet " << first_mismatch->graphlet_id << ": expected "
        << first_mismatch->expected << ", got " << first_mismatch->actual << "\n";
  out << (all_passed() ? "all legs pass" : "cross-check FAILED");
  return out.str();
}

CrossCheckReport cross_check(const SparseAdjacency& g, const RawFrequencyField& fast_raw,
                             const NetFrequencyField& fast_net, OracleOptions opt) {
  if (fast_raw.dictionary() != Dictionary::all() || fast_net.dictionary() != Dictionary::all())
    throw Error("cross_check requires full-dictionary fields");
  const RawFrequencyField oraw = oracle_raw(g, opt);
  const NetFrequencyField onet = oracle_net(g, opt);
  const RawFrequencyField via_u = apply_conversion(onet, full_u16());
  CrossCheckReport rep;
  auto leg = [&](const char* name, const FrequencyField& want, const FrequencyField& got) {
    for (vertex_t v = 0; v < g.num_vertices(); ++v)
      for (std::size_t c = 0; c < 16; ++c)
        if (want.at(v, c) != got.at(v, c)) {
          if (!rep.first_mismatch)
            rep.first_mismatch = CrossCheckReport::Mismatch{name, v, static_cast<int>(c),
                                                            want.at(v, c), got.at(v, c)};
          return false;
        }
    return true;
  };
  rep.raw_ok = leg("fast raw vs oracle raw", oraw, fast_raw);
  rep.net_ok = leg("fast net vs oracle net", onet, fast_net);
  rep.conversion_ok = leg("U*oracle net vs oracle raw", oraw, via_u);
  return rep;
}

count_t count_triangles(const SparseAdjacency& g) {
  count_t t = 0;
  for_each_connected_set(g, [&](const std::array<vertex_t, 4>&, int k, unsigned em) {
    t += k == 3 && em == 0xBu;  // pairs (0,1), (0,2), (1,2) = bits 0, 1, 3
  });
  return t;
}

count_t count_four_cycles(const SparseAdjacency& g) {
  // the three Hamiltonian cycles of a 4-set, as pair masks over kPair*:
  // 0-1-2-3-0, 0-1-3-2-0, 0-2-1-3-0
  constexpr unsigned kCycles[3] = {(1u << 0) | (1u << 3) | (1u << 5) | (1u << 2),
                                   (1u << 0) | (1u << 4) | (1u << 5) | (1u << 1),
                                   (1u << 1) | (1u << 3) | (1u << 4) | (1u << 2)};
  count_t c = 0;
  for_each_connected_set(g, [&](const std::array<vertex_t, 4>&, int k, unsigned em) {
    if (k == 4)
      for (unsigned cyc : kCycles) c += (em & cyc) == cyc;
  });
  return c;
}

count_t count_tetrahedra(const SparseAdjacency& g) {
  count_t q = 0;
  for_each_connected_set(g, [&](const std::array<vertex_t, 4>&, int k, unsigned em) {
    q += k == 4 && em == 63u;
  });
  return q;
}

}  // namespace graphlet
