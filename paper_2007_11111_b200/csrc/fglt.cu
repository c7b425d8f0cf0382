// fglt.cu — host orchestrator + C-ABI (include/fglt.h) of the B200-native
// Fast Graphlet Transform. One CUDA stream per context; all device work is
// stream-ordered; the only host syncs are the small bin-count readbacks and
// the final error word.
//
// Pipeline (reference plan order, proj/src/dictionary.cpp:143-158):
//   prepare   degree relabel (CUB radix sort of n keys + segmented row sort),
//             split/mirror indices, canonical edge list          ["degrees"]
//   sweep A   p2, d7                                              ["two-paths"]
//   K2        per-edge triangle counts C3 (edge-centric, atomics) ["triangles"]
//   sweep B/C c3, d14, d10, p3, d9                                ["three-paths"]
//   K4        4-cycles per vertex (root-centric wedge counting)   ["four-cycle rows"]
//   K5        diamonds + 4-cliques (root bitmaps of G[N+(u)])     ["diamond rows", "tetrahedra"]
//   K6        column fill + raw->net back-substitution, rows written in
//             original vertex order                               ["column fill", "conversion"]
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/fglt.h"
#include "fglt_device.cuh"
#include "fglt_roots.cuh"
#include "fglt_ingest.cuh"
#include "fglt_kernels_api.cuh"

using namespace fglt;

namespace {


#ifndef FGLT_TL_MEM_FRAC
#define FGLT_TL_MEM_FRAC 0.70  // triangle-list pool: at most this share of the free HBM
#endif
#ifndef FGLT_BIG512_MAXOUT
// graphs with max |N+(u)| above this run the 257..1024 root bins on 512
// threads. Always, since the triangle kernel fits 64 registers
// (FGLT_ROOTS_QUADS 1): R-MAT 20 triangles 12.1 -> 11.7 ms (it was +12 % at 80
// registers)
#define FGLT_BIG512_MAXOUT 0
#endif
#ifndef FGLT_FLAT_DMAX
#define FGLT_FLAT_DMAX 0  // graphs with d_max up to this are not relabelled by degree (<= 255); 0 = off:
                          // measured on the SBM (64: DRAM 41 -> 28 GB/step but the 4-cycle classes get uneven roots, 24.4 -> 25.0 ms)
#endif
#ifndef FGLT_TINY_DMAX
#define FGLT_TINY_DMAX 64  // graphs with d_max up to this run tiny roots thread-per-root
#endif
#ifndef FGLT_TL_MIN_RECORDS
#define FGLT_TL_MIN_RECORDS (1ull << 20)  // smaller record bounds: no triangle list
#endif
#ifndef FGLT_MIRROR_SORT_DEG
#define FGLT_MIRROR_SORT_DEG 8  // mean degree from which mirror slots come from a transpose sort
#endif
#ifndef FGLT_C4_CLASS2_THREADS
#define FGLT_C4_CLASS2_THREADS 128
#endif
#ifndef FGLT_C4_CLASS8_THREADS
#define FGLT_C4_CLASS8_THREADS 64
#endif
constexpr int kSmallS = 32;       // roots with |N+(u)| <= 32: warp kernel
constexpr int kBlockS = 1024;     // <= 1024: block kernel, bitmap in smem
constexpr int kWarpHashLog = 9;   // 512-slot table per warp (wc <= 256)
constexpr int kWarpHashLog2 = 11; // 2048-slot table per warp (wc <= 1024)

enum Buf {
  B_RP_IN, B_CI_IN, B_PERM, B_INV, B_NDEG, B_NRP, B_NCI, B_TMP,
  B_SPLIT, B_MIR, B_VEC, B_WORK, B_BINKEY, B_LISTS,
  B_CUB, B_CURSOR, B_TBND, B_BIGROWS, B_HUB, B_HUBBASE, B_ROWOF, B_KEYSOUT, B_GBM, B_RAW, B_NET, B_DICT, B_SMALL, B_RLISTS, B_RKEY,
  B_ING_E, B_ING_K, B_ING_K2, B_ING_RP, B_ING_CI, B_SEND, B_SORTK, B_SORTV,
  B_API0, B_API1, B_API2, B_API3, B_API4, B_API5, B_TB, B_TLREC, B_TLPIECES, B_TLFAIL, B_TBS, B_TBNDS, B_CURSORS, B_TLCHUNKS,
  B_COUNT
};

const char* const kBufName[] = {
  "rp_in", "ci_in", "perm", "inv", "ndeg", "nrp", "nci", "tmp_c3",
  "split", "mir", "vec", "work", "binkey", "lists",
  "cub", "cursor", "tbnd", "bigrows", "hub", "hubbase", "rowof", "keysout", "gbm", "raw", "net",
  "dict", "small", "rlists", "rkey",
  "ing_e", "ing_k", "ing_k2", "ing_rp", "ing_ci", "send", "sortk", "sortv",
  "api0", "api1", "api2", "api3", "api4", "api5", "tb", "tlrec", "tlpieces", "tlfail", "tbs",
  "tbnds", "cursors", "tlchunks"};
static_assert(sizeof(kBufName) / sizeof(kBufName[0]) == B_COUNT, "buffer names");

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  size_t req = 0;     // bytes the current call asked for (<= cap: capacity is kept across calls)
  uint64_t call = 0;  // last call that used this buffer (per-call accounting)
};

// Staging copies of the caller's CSR and of the output tables, and B_VEC (the
// raw columns p2, d7, c3, ... before the fill): the graph and the result
// fields, which the reference's MemoryTracker does not count as auxiliary
// scratch either (proj/include/graphlet/instrumentation.hpp:9-15; its
// per-vertex columns are untracked std::vectors, kernels.cpp:305-419).
inline bool is_staging(int b) {
  return b == B_RP_IN || b == B_CI_IN || b == B_RAW || b == B_NET || b == B_VEC;
}

// Per-vertex vectors, each n u64, in B_VEC.
enum Vec { V_P2, V_D7, V_C3, V_D14, V_D10, V_P3, V_D9, V_C4, V_D13, V_D15, V_COUNT };

struct Plan {
  unsigned mask = 3;
  bool enumerate = false;  // relabel + any enumeration kernel
  bool p2 = false, d7 = false, c3 = false, d14 = false, d10 = false, p3 = false;
  bool d9 = false, c4 = false, d13 = false, d15 = false, dip = false;
  std::vector<std::string> ref_steps;  // reference step names in plan order
};

Plan make_plan(unsigned mask) {
  Plan p;
  mask |= 3u;
  p.mask = mask;
  auto has = [&](int id) { return (mask >> id) & 1u; };
  auto any = [&](std::initializer_list<int> ids) {
    for (int i : ids)
      if (has(i)) return true;
    return false;
  };
  p.p2 = any({2, 5, 6});
  p.p3 = has(5);
  p.d7 = has(7);
  p.dip = any({9, 10, 11});
  p.d9 = p.dip;
  p.d10 = p.dip;
  p.c4 = has(12);
  p.d13 = has(13);
  p.d14 = has(14);
  p.d15 = has(15);
  p.c3 = any({4, 5, 6, 9, 10, 11, 13, 14});
  p.enumerate = p.c3 || p.c4 || p.d13 || p.d15;
  // reference plan (resolve_dependencies, src/dictionary.cpp:143-158), from
  // the shared step table
  for (const auto& st : fglt_tables::kAuxSteps)
    if (mask & st.needed_by) p.ref_steps.push_back(st.name);
  p.ref_steps.push_back("column fill");
  p.ref_steps.push_back("conversion");
  return p;
}

DictInfo make_dict(unsigned mask) {
  DictInfo d;
  std::memset(&d, 0, sizeof(d));
  mask |= 3u;
  d.mask = mask;
  d.k = 0;
  for (int i = 0; i < 16; ++i)
    if (mask & (1u << i)) d.ids[d.k++] = i;
  for (int r = 0; r < d.k; ++r) {
    int t = 0;
    for (int c = r + 1; c < d.k; ++c) {
      unsigned coef = fglt_tables::u16_coef(d.ids[r], d.ids[c]);
      if (coef) {
        d.tail_col[r][t] = c;
        d.tail_coef[r][t] = coef;
        ++t;
      }
    }
    d.ntail[r] = t;
  }
  return d;
}

struct CudaFail {
  int code;
  std::string msg;
};

#define CK(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess)                                                    \
      throw CudaFail{FGLT_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

void set_err(fglt_error* err, int code, int g, int64_t v, const char* fmt, ...) {
  if (!err) return;
  err->code = code;
  err->graphlet_id = g;
  err->vertex = v;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err->msg, sizeof(err->msg), fmt, ap);
  va_end(ap);
}

int group_for(double avg) {
  if (avg < 6) return 4;
  if (avg < 16) return 8;
  if (avg < 48) return 16;
  return 32;
}

}  // namespace

struct fglt_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sms = 148;
  DevBuf buf[B_COUNT];
  size_t scratch_bytes = 0;  // device bytes held by the workspace (all calls)
  // per-call auxiliary scratch (TransformStats::peak_aux_words /
  // largest_aux_alloc_words, reset by begin_call like the reference's
  // MemoryTracker reset in raw_frequencies, src/kernels.cpp:312)
  uint64_t call = 0;
  size_t call_bytes = 0, peak_scratch = 0, largest = 0;
  uint64_t launches = 0, launches_at_call = 0;

  // prepared graph
  int64_t n = 0, nnz = 0, m = 0;
  Plan plan;
  DictInfo dict;
  int lenient = 0;
  const int* rp = nullptr;  // graph the kernels index (relabelled or input)
  const int* ci = nullptr;
  int* perm = nullptr;
  int* inv = nullptr;
  int* split = nullptr;
  int* send = nullptr;  // end of the active part of N+(u)
  int* mir = nullptr;
  u32* C3f = nullptr;
  u64* vec = nullptr;
  DictInfo* d_dict = nullptr;
  u64* d_small = nullptr;  // [0] err key, [1] W, [2] d_max, [3..] bin counts
  bool have_stats = false;
  bool dmax_valid = false;  // dmax is this graph's (set by the stats readbacks)
  uint64_t W = 0, dmax = 0, maxout = 0, nact = 0;

  // last ingest result (fglt_build_csr), on the device
  int64_t ing_n = 0, ing_nnz = 0;

  // root bins by |N+(u)| (shared by the triangle and diamond passes)
  int64_t rb_u0 = -1, rb_u1 = -1;
  std::vector<int> rb_cnt;
  int* rb_lists[9] = {};

  // test hooks (fglt_ctx_set_debug): force one code path for every root
  int force_c4_class = 0, force_c4_parts = 0, force_roots_bin = -1, force_hub = 0;
  // vertex sweeps B/C of a multi-GPU rank: rows r = rows_part (mod rows_parts)
  // only (fglt_stage_local_part); 0 / 1 = every row
  int rows_part = 0, rows_parts = 1;
  bool local_partial = false;  // this call's sweeps B/C were row-partitioned
  int force_row_sort = 0;  // 2: never take the in-register row sort (k_fill_sort)
  // graphs with d_max up to this keep the caller's vertex order among active
  // vertices (k_degree_keys); at most 255 (the dense 4-cycle bands below)
  int flat_dmax = FGLT_FLAT_DMAX;
  bool flat_order() const { return dmax <= (u64)flat_dmax; }
  // triangle list (k_roots_block -> k_diamond_list); tl_mode: 0 auto, 1 off,
  // 2 a tiny pool (test hook: most roots fall back to the probing pass)
  int tl_mode = 0;
  TriList tl;
  int64_t tl_u0 = -1, tl_u1 = -1;  // root range the list was built for
  // hub rows (k_hub_rows): built once per graph by the first root pass
  bool hub_built = false;
  bool big_rows_listed = false;  // list_big_rows
  int* big_rows = nullptr;
  unsigned long long* hub = nullptr;
  int* hub_base = nullptr;
  int hub_hb = 0;

  // timing
  bool timing = false;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  // algorithmic work units of a phase, read after the call's final sync:
  // phase name -> device u64 slot
  std::vector<std::pair<std::string, const u64*>> unit_slots;

  void begin_call() {
    ++call;
    unit_slots.clear();
    call_bytes = peak_scratch = largest = 0;
    launches_at_call = launches;
  }

  // Per-call accounting charges what the call asked for (plus the growth
  // slack when this call allocated), not the capacity an earlier, larger
  // graph left behind.
  template <class T>
  T* ensure(Buf b, size_t count) {
    size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    DevBuf& d = buf[b];
    if (d.call != call) {
      d.call = call;
      d.req = 0;
    }
    if (d.cap < bytes) {
      if (d.p) {
        CK(cudaFreeAsync(d.p, stream));
        scratch_bytes -= d.cap;
      }
      size_t grow = bytes + bytes / 8;
      CK(cudaMallocAsync(&d.p, grow, stream));
      d.cap = grow;
      scratch_bytes += grow;
      bytes = grow;
    }
    if (bytes > d.req) {
      if (!is_staging(b)) call_bytes += bytes - d.req;
      d.req = bytes;
    }
    if (!is_staging(b)) {
      peak_scratch = std::max(peak_scratch, call_bytes);
      largest = std::max(largest, d.req);
    }
    return reinterpret_cast<T*>(d.p);
  }

  u64* V(Vec v) { return vec + (size_t)v * (size_t)std::max<int64_t>(n, 1); }

  void mark(const char* name) {
    if (!timing) return;
    cudaEvent_t ev;
    CK(cudaEventCreate(&ev));
    CK(cudaEventRecord(ev, stream));
    marks.push_back({name, ev});
  }

  int grid(int64_t work, int block, int per_sm = 8) {
    int64_t g = (work + block - 1) / block;
    g = std::min<int64_t>(g, (int64_t)sms * per_sm);
    return (int)std::max<int64_t>(g, 1);
  }

  void launched() { ++launches; }
};

namespace {

void check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw CudaFail{FGLT_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e)};
}

template <class K>
void set_smem(K kernel, size_t bytes) {
  CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

// Long rows (degree > kSweepBig) are listed once per graph for the
// block-per-row sweeps.
void list_big_rows(fglt_ctx* c) {
  if (c->big_rows_listed) return;
  c->big_rows_listed = true;
  int* count = reinterpret_cast<int*>(c->d_small + 5);
  CK(cudaMemsetAsync(count, 0, sizeof(int), c->stream));
  c->big_rows = c->ensure<int>(B_BIGROWS, std::max<int64_t>(c->nnz / (kSweepBig + 1), 1));
  k_list_big_rows<<<c->grid(c->n, 256), 256, 0, c->stream>>>(c->rp, (int)c->n, c->big_rows, count);
  check_launch();
  c->launched();
}

template <int G, class F>
void run_rows(fglt_ctx* c, const F& f) {
  // no row longer than kSweepBig (known d_max): no list, no block-per-row launch
  const bool no_big = c->dmax_valid && c->dmax <= (u64)kSweepBig;
  if (!no_big) list_big_rows(c);
  const int r0 = c->rows_part, rs = std::max(c->rows_parts, 1);
  k_rows_group<G, F><<<c->grid((c->n + rs - 1) / rs * G, 256), 256, 0, c->stream>>>(
      f, c->rp, (int)c->n, r0, rs);
  check_launch();
  c->launched();
  if (no_big) return;
  k_rows_block<F><<<c->sms * 4, kSweepBlock, 0, c->stream>>>(
      f, c->rp, c->big_rows, reinterpret_cast<const int*>(c->d_small + 5), r0, rs);
  check_launch();
  c->launched();
}

template <int G>
void launch_root_work(fglt_ctx* c, u64* wc) {
  RootWork f{c->rp, c->ci, c->split, c->mir, (int)c->nact, wc};
  run_rows<G>(c, f);
}

template <int G>
void launch_sweep_a(fglt_ctx* c) {
  SweepA f{c->rp, c->ci, c->plan.p2 || c->plan.p3 ? c->V(V_P2) : nullptr,
           c->plan.d7 ? c->V(V_D7) : nullptr};
  run_rows<G>(c, f);
}

// phases: 1 = sweep B, 2 = sweep C (needs every row's c3), 3 = both
template <int G>
void launch_sweep_bc(fglt_ctx* c, int phases) {
  if (phases & 1) {
    SweepB fb{c->rp, c->ci, c->C3f, c->mir, (int)c->nact, c->plan.p3 ? c->V(V_P2) : nullptr,
              c->V(V_C3),
              c->plan.d14 ? c->V(V_D14) : nullptr, c->plan.d10 ? c->V(V_D10) : nullptr,
              c->plan.p3 ? c->V(V_P3) : nullptr};
    run_rows<G>(c, fb);
  }
  if ((phases & 2) && c->plan.d9) {
    SweepC fc{c->ci, c->V(V_C3), c->V(V_D9)};
    run_rows<G>(c, fc);
  }
}

template <int G>
void launch_probe_work(fglt_ctx* c, u64* tw) {
  k_probe_work<G><<<c->grid(c->n * G, 256), 256, 0, c->stream>>>(c->split, c->send, c->ci,
                                                                  (int)c->n, c->d_small + 4, tw);
  check_launch();
  c->launched();
}

template <int G>
void launch_c4_hashp(fglt_ctx* c, int g, int block, size_t sm, const int* roots, int nroots,
                     const u64* wc, const u32* parts, int max_log, int* queue, u64* c4) {
  set_smem(k_c4_hashp<G>, sm);
  k_c4_hashp<G><<<g, block, sm, c->stream>>>(c->rp, c->ci, c->split, c->mir, roots, nroots, wc,
                                             parts, max_log, queue, c4);
  check_launch();
  c->launched();
}

#define DISPATCH_G(G, FN, ...)               \
  switch (G) {                               \
    case 4: FN<4>(__VA_ARGS__); break;       \
    case 8: FN<8>(__VA_ARGS__); break;       \
    case 16: FN<16>(__VA_ARGS__); break;     \
    default: FN<32>(__VA_ARGS__); break;     \
  }

template <int G>
void launch_fill_rows(fglt_ctx* c, const int* rp, const int* ci, const int* perm, const int* inv,
                      const int* nrp, int n, int* out, int* row_of) {
  k_fill_rows<G><<<c->grid((int64_t)n * G, 256), 256, 0, c->stream>>>(rp, ci, perm, inv, nrp, n,
                                                                      c->d_small + 4, out, row_of);
  check_launch();
  c->launched();
}

// Low-degree graphs (d_max <= 4 G): rows relabelled, sorted and split by their
// own lane group (k_fill_sort); K = elements per lane.
template <int G>
void launch_fill_sort(fglt_ctx* c, const int* rp, const int* ci, const int* perm, const int* inv,
                      const int* nrp, int n, int* out, int* split, int* send) {
  const int K = (int)((c->dmax + G - 1) / G);
  const int g = c->grid((int64_t)n * G, 256);
  u64* nact_p = c->d_small + 4;
  u64* maxout = c->d_small + 3;
  if (K <= 1)
    k_fill_sort<G, 1><<<g, 256, 0, c->stream>>>(rp, ci, perm, inv, nrp, n, nact_p, out, split, send, maxout);
  else if (K == 2)
    k_fill_sort<G, 2><<<g, 256, 0, c->stream>>>(rp, ci, perm, inv, nrp, n, nact_p, out, split, send, maxout);
  else
    k_fill_sort<G, 4><<<g, 256, 0, c->stream>>>(rp, ci, perm, inv, nrp, n, nact_p, out, split, send, maxout);
  check_launch();
  c->launched();
}

template <int G>
void launch_mirror(fglt_ctx* c, const int* split, const int* send, int n, int* mir) {
  k_mirror<G><<<c->grid((int64_t)n * G, 256), 256, 0, c->stream>>>(c->rp, c->ci, split, send, n,
                                                                   mir);
  check_launch();
  c->launched();
}

// Graph totals of the INPUT row pointer (k_graph_stats): W, d_max, n_active.
// Read once, early: d_max picks the relabel path; the device keeps working on
// the degree sort while the host waits.
void read_input_stats(fglt_ctx* c) {
  u64 h[4];
  CK(cudaMemcpyAsync(h, c->d_small + 1, 32, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->W = h[0];
  c->dmax = h[1];
  c->dmax_valid = true;
  c->nact = h[3];
}

// ------------------------------------------------------------------ prepare
void prepare(fglt_ctx* c, const int* d_rp, const int* d_ci, int64_t n, int64_t nnz,
             unsigned mask, int lenient) {
  c->n = n;
  c->nnz = nnz;
  c->m = nnz / 2;
  c->plan = make_plan(mask);
  c->dict = make_dict(mask);
  c->lenient = lenient;
  c->d_dict = c->ensure<DictInfo>(B_DICT, 1);
  CK(cudaMemcpyAsync(c->d_dict, &c->dict, sizeof(DictInfo), cudaMemcpyHostToDevice, c->stream));
  c->d_small = c->ensure<u64>(B_SMALL, 64);
  CK(cudaMemsetAsync(c->d_small, 0, 64 * sizeof(u64), c->stream));
  {
    u64 init = ~0ull;
    CK(cudaMemcpyAsync(c->d_small, &init, 8, cudaMemcpyHostToDevice, c->stream));
  }
  const int N = (int)n;
  c->vec = c->ensure<u64>(B_VEC, (size_t)V_COUNT * std::max<int64_t>(n, 1));
  CK(cudaMemsetAsync(c->vec, 0, (size_t)V_COUNT * std::max<int64_t>(n, 1) * 8, c->stream));
  c->perm = c->inv = nullptr;
  c->rows_part = 0;
  c->rows_parts = 1;
  c->local_partial = false;
  c->rb_u0 = c->rb_u1 = -1;  // graph changed: root bins are stale
  c->hub_built = false;
  c->big_rows_listed = false;
  c->rb_cnt.clear();
  c->rp = d_rp;
  c->ci = d_ci;
  c->have_stats = false;
  c->dmax_valid = false;
  if (n > 0) {
    k_graph_stats<<<c->grid(n, 256, 4), 256, 0, c->stream>>>(d_rp, N, c->d_small + 1);
    check_launch();
    c->launched();
  }
  if (!c->plan.enumerate || n == 0) return;

  // ---- degree relabel: rank by (degree, id) = stable sort of the ids by
  // the degree key (k_degree_keys), over the key's live bits only. Every sort
  // here runs on cub::DoubleBuffer pairs of our own arrays: no hidden
  // (keys + values)-sized temporary.
  // The sort's four n-int arrays are buffers nothing has written yet: keys in
  // (nrp, ndeg), ids in (split, perm); if the sorted ids land in perm itself,
  // k_perm's copy is the identity.
  int* perm = c->ensure<int>(B_PERM, n);
  int* inv = c->ensure<int>(B_INV, n);
  int* ndeg = c->ensure<int>(B_NDEG, n + 1);
  int* nrp = c->ensure<int>(B_NRP, n + 1);
  int* split = c->ensure<int>(B_SPLIT, n);
  int* send = c->ensure<int>(B_SEND, n);
  int key_bits = 1;
  while (key_bits < 31 && ((int64_t)1 << key_bits) <= n + 1) ++key_bits;
  k_degree_keys<<<c->grid(n, 256), 256, 0, c->stream>>>(d_rp, N, nrp, split, c->d_small + 1,
                                                        (u64)c->flat_dmax);
  check_launch();
  c->launched();
  int id_bits = 1;
  while (id_bits < 31 && ((int64_t)1 << id_bits) < n) ++id_bits;
  size_t tmp_bytes = 0, t2 = 0, t3 = 0;
  {
    cub::DoubleBuffer<int> dk(nrp, ndeg), dv(split, perm);
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, N, 0, key_bits, c->stream));
    CK(cub::DeviceScan::ExclusiveSum(nullptr, t2, ndeg, nrp, N + 1, c->stream));
    CK(cub::DeviceRadixSort::SortPairs(nullptr, t3, dk, dv, (int)std::max<int64_t>(nnz, 1), 0,
                                       id_bits, c->stream));  // size query only
  }
  tmp_bytes = std::max(tmp_bytes, std::max(t2, t3));
  void* cub_tmp = c->ensure<unsigned char>(B_CUB, tmp_bytes);
  size_t tb = c->buf[B_CUB].cap;
  const int* sorted_ids = nullptr;
  {
    cub::DoubleBuffer<int> dk(nrp, ndeg), dv(split, perm);
    CK(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, dk, dv, N, 0, key_bits, c->stream));
    sorted_ids = dv.Current();
  }
  c->launched();
  read_input_stats(c);  // overlaps the degree sort
  CK(cudaMemsetAsync(ndeg + n, 0, sizeof(int), c->stream));
  k_perm<<<c->grid(n, 256), 256, 0, c->stream>>>(sorted_ids, d_rp, N, perm, inv, ndeg);
  check_launch();
  c->launched();
  tb = c->buf[B_CUB].cap;
  CK(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, ndeg, nrp, N + 1, c->stream));
  c->launched();
  const int G = group_for((double)nnz / (double)std::max<int64_t>(n, 1));
  int* tmp = c->ensure<int>(B_TMP, std::max<int64_t>(nnz, 1));  // fill scratch, then C3
  int* nci = c->ensure<int>(B_NCI, std::max<int64_t>(nnz, 1) + 4);  // +4: 16-byte tail reads
  int* free_vals = nullptr;   // nnz-int arrays the row sort leaves free
  int* free_keys = nullptr;
  const bool row_sort = c->force_row_sort != 2 && (c->dmax <= (u64)(4 * G));
  if (row_sort) {
    DISPATCH_G(G, launch_fill_sort, c, d_rp, d_ci, perm, inv, nrp, N, nci, split, send);
  } else {
    int* row_of = c->ensure<int>(B_ROWOF, std::max<int64_t>(nnz, 1) + 4);
    int* keys_out = c->ensure<int>(B_KEYSOUT, std::max<int64_t>(nnz, 1));
    DISPATCH_G(G, launch_fill_rows, c, d_rp, d_ci, perm, inv, nrp, N, tmp, row_of);
    if (nnz > 0) {  // stable sort by neighbour id: rows come out sorted (see k_fill_rows)
      cub::DoubleBuffer<int> dk(tmp, keys_out), dv(row_of, nci);
      tb = c->buf[B_CUB].cap;
      CK(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, dk, dv, (int)nnz, 0, id_bits, c->stream));
      c->launched();
      if (dv.Current() != nci) std::swap(nci, row_of);  // the sorted rows may land in either
    }
    free_vals = row_of;
    free_keys = keys_out;
  }
  c->perm = perm;
  c->inv = inv;
  c->rp = nrp;
  c->ci = nci;

  // ---- split / mirror
  if (!row_sort) {
    k_split<<<c->grid(n, 256), 256, 0, c->stream>>>(c->rp, c->ci, N, c->d_small + 4, split, send,
                                                    c->d_small + 3);
    check_launch();
    c->launched();
  }
  int* mir = c->ensure<int>(B_MIR, std::max<int64_t>(nnz, 1));
  const bool sort_mirror = nnz >= FGLT_MIRROR_SORT_DEG * n;  // else per-edge binary searches
  if (nnz > 0 && !sort_mirror) {
    DISPATCH_G(G, launch_mirror, c, split, send, N, mir);
  } else if (nnz > 0) {
    // mirror positions by a second stable transpose: the sorted CSR read
    // r-major as (key = neighbour y, value = own position j) sorts into
    // y-major order with r ascending, i.e. the value landing at j' (the slot
    // of (y, r)) is j, the slot of (r, y). Keys: a copy of the column array
    // (in the C3 buffer, zeroed later anyway).
    if (!free_vals) free_vals = c->ensure<int>(B_ROWOF, std::max<int64_t>(nnz, 1) + 4);
    if (!free_keys) free_keys = c->ensure<int>(B_KEYSOUT, std::max<int64_t>(nnz, 1));
    k_iota_copy<<<c->grid(nnz, 256), 256, 0, c->stream>>>(free_vals, tmp, c->ci, nnz);
    check_launch();
    c->launched();
    cub::DoubleBuffer<int> dk(tmp, free_keys), dv(free_vals, mir);
    tb = c->buf[B_CUB].cap;
    CK(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, dk, dv, (int)nnz, 0, id_bits, c->stream));
    c->launched();
    mir = dv.Current();
  }
  c->split = split;
  c->send = send;
  c->mir = mir;
  c->C3f = reinterpret_cast<u32*>(tmp);  // B_TMP is dead after the sorts
}

void read_graph_stats(fglt_ctx* c) {
  u64 h[4];
  CK(cudaMemcpyAsync(h, c->d_small + 1, 32, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->W = h[0];
  c->dmax = h[1];
  c->dmax_valid = true;
  c->maxout = h[2];
  c->nact = h[3];
  c->have_stats = true;
}

void sweep_a(fglt_ctx* c) {
  if (c->n == 0) return;
  if (!(c->plan.p2 || c->plan.p3 || c->plan.d7)) return;
  const int G = group_for((double)c->nnz / (double)c->n);
  DISPATCH_G(G, launch_sweep_a, c);
}


// Vertex sweeps over the per-edge triangle counts. The counts stay at the
// canonical slots (SweepB reads lower neighbours through mir); the per-kernel
// API, which hands C3 out in CSR order, mirrors them first.
void local_sweeps(fglt_ctx* c, bool mirror_c3 = false, int phases = 3) {
  if (!c->plan.c3 || c->n == 0) return;
  if (mirror_c3 && c->m > 0) {
    k_c3_mirror<<<c->grid((int64_t)c->nact * 8, 256), 256, 0, c->stream>>>(
        c->split, c->send, c->mir, (int)c->nact, c->C3f);
    check_launch();
    c->launched();
  }
  const int G = group_for((double)c->nnz / (double)c->n);
  DISPATCH_G(G, launch_sweep_bc, c, phases);
}

// Bin roots [u0,u1) by key into compact lists; returns the counts (host
// sync). The kernel that wrote the keys tallied the bins into bin_counts(c)
// (zeroed by bin_counts_reset before it ran).
int* bin_counts(fglt_ctx* c) { return reinterpret_cast<int*>(c->d_small + 16); }

void bin_counts_reset(fglt_ctx* c) {
  CK(cudaMemsetAsync(bin_counts(c), 0, 10 * sizeof(int), c->stream));  // slots 16..20
}

std::vector<int> bin_roots(fglt_ctx* c, const u32* key, int64_t u0, int64_t u1,
                           const std::vector<u64>& thr, int** lists, Buf which = B_LISTS) {
  const int nb = (int)thr.size() + 1;
  if (nb > 9) throw CudaFail{FGLT_E_CUDA, "internal: at most 9 root bins"};
  std::vector<int> h(9);
  CK(cudaMemcpyAsync(h.data(), bin_counts(c), 9 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  h.resize(nb);
  BinThr T;
  BinBases B;
  for (int b = 0; b < 8; ++b) T.thr[b] = b < (int)thr.size() ? thr[b] : ~0ull;
  T.nbins = nb;
  int64_t total = 0;
  for (int b = 0; b < 9; ++b) {
    B.base[b] = (int)total;
    if (b < nb) total += h[b];
  }
  int* lst = c->ensure<int>(which, (size_t)std::max<int64_t>(total, 1));
  for (int b = 0; b < nb; ++b) lists[b] = lst + B.base[b];
  if (total > 0) {
    int* cursors = reinterpret_cast<int*>(c->d_small + 44);  // slots 44..48
    CK(cudaMemsetAsync(cursors, 0, 10 * sizeof(int), c->stream));
    k_bin<<<c->grid(u1 - u0, 256), 256, 0, c->stream>>>(key, (int)u0, (int)u1, T, B, cursors, lst);
    check_launch();
    c->launched();
  }
  return h;
}


__global__ void k_outdeg_key(const int* __restrict__ send, const int* __restrict__ split, int n,
                             u32* __restrict__ key, u32 force_key, int u0, int u1, BinThr T,
                             int* __restrict__ counts) {
  int tally = 0;
  const int lane = threadIdx.x & 31;
  for (int ub = blockIdx.x * blockDim.x + threadIdx.x - lane; ub < n;
       ub += gridDim.x * blockDim.x) {  // warp-uniform trip count (bin_tally votes)
    const int u = ub + lane;
    u32 k = 0;
    if (u < n) {
      const int s = send[u] - split[u];
      k = s >= 2 ? (u32)s : 0u;
      // test hook: push roots into a larger bin (a bin's kernel handles any s
      // below its cap, so forcing upward is always valid)
      if (k && force_key && force_key > k) k = force_key;
      key[u] = k;
    }
    bin_tally(u >= u0 && u < u1 ? bin_of(k, T) : -1, T.nbins, tally);
  }
  bin_tally_flush(tally, T.nbins, counts);
}

#ifndef FGLT_SPLIT_BIG
#define FGLT_SPLIT_BIG 0  // big-tile packed roots as (root, tile) items too
#endif
#ifndef FGLT_SLAB_BLOCKS_PER_SM
#define FGLT_SLAB_BLOCKS_PER_SM 1  // resident global-slab root blocks per SM (|S| > 1024)
#endif
#ifndef FGLT_SLAB_THREADS
#define FGLT_SLAB_THREADS 1024  // block threads of the global-slab root bin (|S| > 1024); R-MAT 23 triangles: 2 x 256: 216, 2 x 512: 210, 1 x 1024: 206 ms
#endif
constexpr int kSlabThreads = FGLT_SLAB_THREADS;
#ifndef FGLT_DLIST_NT
#define FGLT_DLIST_NT 256  // block threads of the diamond-list kernel
#endif
#ifndef FGLT_BIN1_NT
#define FGLT_BIN1_NT 64   // block threads of root bin 1 (64, 128 or 256)
#define FGLT_BIN2_NT 128  // ... and of bin 2
#endif
#ifndef FGLT_BIN1
#define FGLT_BIN1 128  // |S| cap of the 64-thread root bin
#define FGLT_BIN2 256  // |S| cap of the 128-thread root bin
#define FGLT_BIN3 512
#endif
// root bins by |N+(u)|: 0 tiny (thread per root on low-degree graphs, else
// warp), 1 warp, 2..5 shared-memory block bins, 6 global slab
constexpr u64 kRootThr[] = {(u64)kRootsTiny, (u64)kSmallS, FGLT_BIN1, FGLT_BIN2, FGLT_BIN3,
                            (u64)kBlockS};
constexpr int kFirstBlockBin = 2;

template <class T>
__global__ void k_gather_keys(const int* __restrict__ list, int cnt, const T* __restrict__ w,
                              u64* __restrict__ keys) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x)
    keys[i] = w[list[i]];
}

// Order a root list by work, largest first (LPT for the dynamic queues).
// Keys are < 2^bits (radix passes only over the live bits).
template <class T>
void sort_by_work_desc(fglt_ctx* c, int* list, int cnt, const T* w, int bits = 64) {
  if (cnt < 2) return;
  bits = std::max(1, std::min(bits, 64));
  u64* k = c->ensure<u64>(B_SORTK, 2 * (size_t)cnt);
  int* v = c->ensure<int>(B_SORTV, (size_t)cnt);
  k_gather_keys<T><<<c->grid(cnt, 256), 256, 0, c->stream>>>(list, cnt, w, k);
  check_launch();
  c->launched();
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, k, k + cnt, list, v, cnt, 0, bits,
                                               c->stream));
  void* tmp = c->ensure<unsigned char>(B_CUB, tb);
  tb = c->buf[B_CUB].cap;
  CK(cub::DeviceRadixSort::SortPairsDescending(tmp, tb, k, k + cnt, list, v, cnt, 0, bits,
                                               c->stream));
  c->launched();
  CK(cudaMemcpyAsync(list, v, (size_t)cnt * 4, cudaMemcpyDeviceToDevice, c->stream));
}

// Bin roots [u0,u1) by |N+(u)| (>= 2) once; both root passes reuse the lists.
void build_hubs(fglt_ctx* c) {
  if (c->hub_built) return;
  c->hub_built = true;
  c->hub = nullptr;
  const int64_t nact = (int64_t)c->nact;
  if (c->force_hub == 1 || nact < 2) return;
  const int R = (int)std::min<int64_t>(nact, kHubMax);
  c->hub_hb = (int)(nact - R);
  if (c->force_hub != 2 && c->dmax < (u64)kHubMinDegree) return;  // no hubs: no readback
  if (c->force_hub != 2) {  // only graphs with real hubs: the smallest hub's degree
    int h[2];
    CK(cudaMemcpyAsync(h, c->rp + c->hub_hb, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (h[1] - h[0] < kHubMinDegree) return;
  }
  int* hw = c->ensure<int>(B_HUBBASE, 2 * (size_t)(R + 1));
  int* base = hw + (R + 1);
  k_hub_words<<<c->grid(R + 1, 256), 256, 0, c->stream>>>(R, hw);
  check_launch();
  c->launched();
  size_t tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, hw, base, R + 1, c->stream));
  void* tmp = c->ensure<unsigned char>(B_CUB, tb);
  tb = c->buf[B_CUB].cap;
  CK(cub::DeviceScan::ExclusiveSum(tmp, tb, hw, base, R + 1, c->stream));
  c->launched();
  // words = sum_i ceil((R-1-i)/32), computed on the host
  size_t words = 0;
  for (int i = 0; i < R; ++i) words += (size_t)((R - 1 - i + 31) >> 5);
  c->hub = c->ensure<unsigned long long>(B_HUB, std::max<size_t>(words, 1));
  k_hub_rows<<<c->grid((int64_t)R * 32, 256), 256, 0, c->stream>>>(c->ci, c->split, c->send,
                                                                  c->hub_hb, R, base, c->hub);
  check_launch();
  c->launched();
  c->hub_base = base;
}

void root_bins(fglt_ctx* c, int64_t u0, int64_t u1) {
  build_hubs(c);
  if (c->rb_u0 == u0 && c->rb_u1 == u1 && !c->rb_cnt.empty()) return;
  u32* key = c->ensure<u32>(B_RKEY, (size_t)std::max<int64_t>(c->n, 1));
  static const u32 kForceKey[] = {0, 33, 129, 257, 513, 1025};
  const u32 fk = (c->force_roots_bin > 0 && c->force_roots_bin < 6) ? kForceKey[c->force_roots_bin] : 0;
  const std::vector<u64> thr(std::begin(kRootThr), std::end(kRootThr));
  BinThr T;
  for (int b = 0; b < 8; ++b) T.thr[b] = b < (int)thr.size() ? thr[b] : ~0ull;
  T.nbins = (int)thr.size() + 1;
  bin_counts_reset(c);
  k_outdeg_key<<<c->grid(c->n, 256), 256, 0, c->stream>>>(c->send, c->split, (int)c->n, key, fk,
                                                         (int)u0, (int)u1, T, bin_counts(c));
  check_launch();
  c->launched();
  c->rb_cnt = bin_roots(c, key, u0, u1, thr, c->rb_lists, B_RLISTS);
  // keys are |N+(u)| <= max out-degree (or a forced bin key <= 1025)
  const int kbits = 64 - __builtin_clzll(std::max<u64>(std::max<u64>(c->maxout, 1025), 1));
  for (int b = kFirstBlockBin; b < (int)c->rb_cnt.size(); ++b)
    sort_by_work_desc(c, c->rb_lists[b], c->rb_cnt[b], key, kbits);
  c->rb_u0 = u0;
  c->rb_u1 = u1;
}

// One root-centric pass over the binned roots: MODE 0 = triangle pass (C3
// atomics, plus 4-cliques when requested), MODE 1 = diamond pass (needs final C3).
template <bool kC3, bool kD13, bool kD15>
void roots_pass(fglt_ctx* c) {
  if (!c->have_stats)  // the bins are sized by max |N+(u)|: never guess
    throw CudaFail{FGLT_E_CUDA, "internal: graph stats not read before a root pass"};
  u64* d13 = c->V(V_D13);
  u64* d15 = c->V(V_D15);
  const std::vector<int>& cnt = c->rb_cnt;
  int** lists = c->rb_lists;
  int* queues = reinterpret_cast<int*>(c->d_small + 60);  // one dynamic queue per bin
  CK(cudaMemsetAsync(queues, 0, 8 * sizeof(int), c->stream));
  // thread-per-root for the tiny bin of low-degree graphs only (on power-law
  // graphs the members' probe lists are long: the warp kernel wins there)
  const bool tiny = c->dmax <= (u64)FGLT_TINY_DMAX;
  for (int b = 0; b < kFirstBlockBin; ++b) {
    if (cnt[b] == 0) continue;
    if (b == 0 && tiny) {
      k_roots_tiny<kC3, kD13, kD15><<<c->grid(cnt[0], 256), 256, 0, c->stream>>>(
          c->rp, c->ci, c->split, c->send, c->C3f, lists[0], cnt[0], d13, d15);
    } else {
      const int wpb = 8;
      const size_t sm = (size_t)wpb * (32 * 8 + kRootsWarpInts * 4);
      const int g = c->grid((int64_t)cnt[b] * 32, wpb * 32);
      k_roots_warp<kC3, kD13, kD15><<<g, wpb * 32, sm, c->stream>>>(
          c->rp, c->ci, c->split, c->send, c->C3f, lists[b], cnt[b], d13, d15, c->hub,
          c->hub_base, c->hub_hb, c->force_hub == 2, c->tl);
    }
    check_launch();
    c->launched();
  }
  for (int b = kFirstBlockBin; b < (int)cnt.size(); ++b) {
    if (cnt[b] == 0) continue;
    const bool global = b == (int)cnt.size() - 1;  // s > kBlockS
    RootsLayout L;
    L.s_cap = global ? (int)c->maxout : (int)std::min<u64>(kRootThr[b], std::max<u64>(c->maxout, 33));
    L.hlog = 6;
    while ((1 << L.hlog) < FGLT_ROOT_HASH_FACTOR * L.s_cap) ++L.hlog;
    L.hcap = 1 << L.hlog;
    // block size follows |S|: 64 threads for |S| <= 128, 128 for <= 256, else 256
    // graphs with roots beyond the shared-memory bins have long probe lists:
    // their 257..1024 bins take 512-thread blocks (R-MAT 23 -7 %; R-MAT 20,
    // max |S| 777, keeps 256: +12 % otherwise)
    const int big_nt = c->maxout > (u64)FGLT_BIG512_MAXOUT ? 512 : kRootsThreads;
    const int nt = global ? kSlabThreads
                          : (b == kFirstBlockBin ? FGLT_BIN1_NT
                                                 : b == kFirstBlockBin + 1 ? FGLT_BIN2_NT : big_nt);
    L.nwarps = nt / 32;
    L.stride_cap = bitmap_stride((L.s_cap + 31) / 32);
    size_t sm = L.bytes_core();
    unsigned char* slab = nullptr;
    long long slab_stride = 0;
    int g = std::min(cnt[b], c->sms * std::max(1, 8 * kRootsThreads / nt));
#define FGLT_ROOTS_LAUNCH(GLOBAL, NT)                                                              \
  do {                                                                                             \
    set_smem(k_roots_block<kC3, kD13, kD15, GLOBAL, NT>, sm);                                      \
    k_roots_block<kC3, kD13, kD15, GLOBAL, NT><<<g, NT, sm, c->stream>>>(                         \
        c->rp, c->ci, c->split, c->send, c->C3f, lists[b], cnt[b], L, slab, slab_stride,           \
        queues + b, d13, d15, c->hub, c->hub_base, c->hub_hb, c->force_hub == 2, c->tl);           \
  } while (0)
    if (global) {
      slab_stride = (long long)((L.bytes_aux() + 255) & ~(size_t)255);
      const long long fit = std::max<long long>(1, (4ll << 30) / slab_stride);
      int occ = 1;  // resident blocks per SM (shared memory holds the per-member arrays)
      set_smem(k_roots_block<kC3, kD13, kD15, true, kSlabThreads>, sm);
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &occ, k_roots_block<kC3, kD13, kD15, true, kSlabThreads>, kSlabThreads, sm));
      g = (int)std::min<long long>(
          {(long long)cnt[b], (long long)c->sms * std::max(1, std::min(occ, FGLT_SLAB_BLOCKS_PER_SM)), fit});
      slab = c->ensure<unsigned char>(B_GBM, (size_t)g * (size_t)slab_stride);
      FGLT_ROOTS_LAUNCH(true, kSlabThreads);
    } else {
      sm += L.bytes_aux();
      if (nt == 64) FGLT_ROOTS_LAUNCH(false, 64);
      else if (nt == 128) FGLT_ROOTS_LAUNCH(false, 128);
      else if (nt == 512) FGLT_ROOTS_LAUNCH(false, 512);
      else FGLT_ROOTS_LAUNCH(false, kRootsThreads);
    }
#undef FGLT_ROOTS_LAUNCH
    check_launch();
    c->launched();
  }
}

// Triangle-list pool for the roots [u0,u1) (see TriList): sized by the
// C(|S|,2) bound plus one grab per block, capped at FGLT_TL_MEM_FRAC (70%) of free memory.
void setup_trilist(fglt_ctx* c, int64_t u0, int64_t u1) {
  c->tl = TriList{};
  const Plan& P = c->plan;
  if (!(P.c3 && P.d13) || c->tl_mode == 1 || u1 <= u0) return;
  unsigned long long* d_bound = reinterpret_cast<unsigned long long*>(c->d_small + 24);
  CK(cudaMemsetAsync(d_bound, 0, 4 * sizeof(u64), c->stream));
  k_trilist_bound<<<c->grid(u1 - u0, 256), 256, 0, c->stream>>>(c->split, c->send, c->ci,
                                                               (int)u0, (int)u1, d_bound);
  check_launch();
  c->launched();
  unsigned long long bound = 0;
  CK(cudaMemcpyAsync(&bound, d_bound, 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  // small graphs: the probing diamond pass is cheap, a pool is not worth it
  if (bound < FGLT_TL_MIN_RECORDS && c->tl_mode != 2) return;
  // slack for the reservations the launched blocks and warps hold at once
  // (each grabs >= kTriListChunk / kTriListWarpChunk records): bounded by the
  // grids roots_pass actually launches, so the pool follows the graph size
  unsigned long long blocks = 0, warps = 0;
  if (!c->rb_cnt.empty()) {
    for (int b = 0; b < kFirstBlockBin; ++b)
      warps += std::min<unsigned long long>(c->rb_cnt[b], (unsigned long long)c->sms * 64);
    for (size_t b = kFirstBlockBin; b < c->rb_cnt.size(); ++b)
      blocks += std::min<unsigned long long>(c->rb_cnt[b], (unsigned long long)c->sms * 32);
  }
  unsigned long long cap = bound + blocks * kTriListChunk + warps * kTriListWarpChunk;
  if (cap * 8 > c->buf[B_TLREC].cap) {  // growing: stay within FGLT_TL_MEM_FRAC of free memory
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    cap = std::min<unsigned long long>(
        cap, (unsigned long long)(FGLT_TL_MEM_FRAC * (double)(free_b + c->buf[B_TLREC].cap)) / 8);
  }
  if (c->tl_mode == 2) cap = 4096;
  if (cap < 1024) return;
  TriList t;
  t.rec = c->ensure<uint2>(B_TLREC, cap);
  t.cap = cap;
  t.top = d_bound + 1;
  t.npieces = reinterpret_cast<unsigned*>(d_bound + 2);
  t.pieces_cap = (unsigned)std::min<int64_t>(2 * (u1 - u0) + c->nnz / 32 + 1024, 1ll << 31);
  t.pieces = c->ensure<TriPiece>(B_TLPIECES, t.pieces_cap);
  t.fail = c->ensure<unsigned char>(B_TLFAIL, (size_t)c->n);
  CK(cudaMemsetAsync(t.fail, 0, (size_t)c->n, c->stream));
  t.chunks_cap = (unsigned)std::min<unsigned long long>(cap / kTriListWarpChunk + warps + 1024,
                                                        1ull << 31);
  t.chunks = c->ensure<TriChunk>(B_TLCHUNKS, t.chunks_cap);
  t.nchunks = reinterpret_cast<unsigned*>(d_bound + 3);
  c->tl = t;
}

// Diamonds of the listed roots (the rest take the probing pass).
void diamond_list(fglt_ctx* c) {
  if (!c->tl.rec) return;
  constexpr int NT = FGLT_DLIST_NT;
  const size_t sm = (size_t)std::min<u64>(std::max<u64>(c->maxout, 1), kTriListMaxS) * 8;
  set_smem(k_diamond_list<NT>, sm);
  int occ = 1;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_diamond_list<NT>, NT, sm));
  int* next = reinterpret_cast<int*>(c->d_small + 28);
  CK(cudaMemsetAsync(next, 0, sizeof(int), c->stream));
  k_diamond_list<NT><<<c->sms * std::max(occ, 1), NT, sm, c->stream>>>(
      c->tl.pieces, c->tl.npieces, c->tl.pieces_cap, c->tl.rec, c->rp, c->ci, c->split, c->send,
      c->C3f, c->tl.fail, next, c->V(V_D13));
  check_launch();
  c->launched();
  k_diamond_wlist<<<c->sms * 8, 256, 0, c->stream>>>(c->tl.chunks, c->tl.nchunks,
                                                     c->tl.chunks_cap, c->tl.rec, c->rp, c->ci,
                                                     c->split, c->send, c->C3f, c->V(V_D13));
  check_launch();
  c->launched();
}

// Triangle pass over roots [u0,u1): per-edge C3 (and d15 when requested).
void triangles(fglt_ctx* c, int64_t u0, int64_t u1) {
  const Plan& P = c->plan;
  c->tl = TriList{};
  if (!(P.c3 || P.d15) || c->n == 0) return;
  if (P.c3) CK(cudaMemsetAsync(c->C3f, 0, (size_t)std::max<int64_t>(c->nnz, 1) * 4, c->stream));
  root_bins(c, u0, u1);
  setup_trilist(c, u0, u1);
  c->tl_u0 = u0;
  c->tl_u1 = u1;
  c->mark("triangle pass:start");
  if (P.c3 && P.d15) roots_pass<true, false, true>(c);
  else if (P.c3) roots_pass<true, false, false>(c);
  else roots_pass<false, false, true>(c);
  c->mark("triangle pass:end");
}

void roots(fglt_ctx* c, int64_t u0, int64_t u1) {
  const Plan& P = c->plan;
  if (c->n == 0 || !(P.c4 || P.d13)) return;
  u64* work = c->ensure<u64>(B_WORK, 2 * (size_t)c->n);  // wc (u64) | class, parts (u32 each)
  u64* wc = work;
  u32* cls = reinterpret_cast<u32*>(work + c->n);
  u32* parts = cls + c->n;
  int* lists[9];
  if (P.c4) {
    const int G = group_for((double)c->nnz / (double)c->n);
    DISPATCH_G(G, launch_root_work, c, wc);
    // degree bands of the dense counters (4 / 8 / 16-or-32 bits)
    int bands[3] = {0, 0, 0};
    if (c->nact > 0 && c->dmax <= 15) {  // every active id in the 4-bit band: no readback
      bands[0] = bands[1] = bands[2] = (int)c->nact;
    } else if (c->nact > 0 && c->flat_order()) {  // ids not in degree order: one 8-bit band
      bands[0] = 0;
      bands[1] = bands[2] = (int)c->nact;
    } else if (c->nact > 0) {
      int* d_b = reinterpret_cast<int*>(c->d_small + 41);
      k_degree_bands<<<1, 32, 0, c->stream>>>(c->rp, (int)c->nact, d_b);
      check_launch();
      c->launched();
      CK(cudaMemcpyAsync(bands, d_b, sizeof(bands), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
    unsigned long long* cw = reinterpret_cast<unsigned long long*>(c->d_small + 32);
    CK(cudaMemsetAsync(cw, 0, 2 * sizeof(u64), c->stream));
    c->unit_slots.push_back({"c4 dense", c->d_small + 32});
    c->unit_slots.push_back({"c4 classes", c->d_small + 33});
    c->mark("c4 classes:start");
    bin_counts_reset(c);
    k_c4_class<<<c->grid(u1 - u0, 256), 256, 0, c->stream>>>(
        c->rp, c->split, wc, (int)u0, (int)u1, bands[0], bands[1], bands[2], cls, parts,
        c->force_c4_class, c->force_c4_parts, cw, bin_counts(c));
    check_launch();
    c->launched();
    std::vector<int> cnt = bin_roots(c, cls, u0, u1, {1, 2, 3, 4, 5, 6, 7, 8}, lists);
    // wc(u) <= W = sum of squared degrees
    const int wbits = 64 - __builtin_clzll(std::max<u64>(c->W, 1));
    for (int bb = 3; bb <= 6; ++bb) sort_by_work_desc(c, lists[bb], cnt[bb], wc, wbits);
    int* queues = reinterpret_cast<int*>(c->d_small + 56);  // dynamic root queues
    CK(cudaMemsetAsync(queues, 0, 8 * sizeof(int), c->stream));
    c->mark("c4 classes:end");
    c->mark("four-cycle rows:start");
    c->mark("c4 hash:start");
    u64* c4 = c->V(V_C4);
    if (cnt[8] > 0) {  // class 9: thread per root, at most kC4Tiny wedges
      k_c4_tiny<<<c->grid(cnt[8], 256), 256, 0, c->stream>>>(c->rp, c->ci, c->split, c->mir,
                                                             lists[8], cnt[8], wc, c4);
      check_launch();
      c->launched();
    }
    if (cnt[0] > 0) {  // class 1: warp tables of 512 slots
      const int wpb = 8;
      const size_t sm = (size_t)wpb * ((1 << kWarpHashLog) * 2 + 100) * 4;
      k_c4_warp<kWarpHashLog><<<c->grid((int64_t)cnt[0] * 32, wpb * 32), wpb * 32, sm, c->stream>>>(
          c->rp, c->ci, c->split, c->mir, lists[0], cnt[0], wc, c4);
      check_launch();
      c->launched();
    }
    if (cnt[1] > 0) {  // class 2: block-flattened tables of <= 2048 slots
      constexpr int NT2 = FGLT_C4_CLASS2_THREADS;
      const size_t sm = (size_t)(1 << kWarpHashLog2) * 8;
      set_smem(k_c4_block<NT2, true>, sm);
      int occ = 1;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_c4_block<NT2, true>, NT2, sm));
      const int g = std::min(cnt[1], c->sms * std::max(occ, 1));
      k_c4_block<NT2, true><<<g, NT2, sm, c->stream>>>(c->rp, c->ci, c->split, c->mir, lists[1], cnt[1],
                                                wc, parts, kWarpHashLog2, queues + 4, c4);
      check_launch();
      c->launched();
    }
    if (cnt[7] > 0) {  // class 8: block-flattened tables of <= 1024 slots
      constexpr int NT8 = FGLT_C4_CLASS8_THREADS;
      const size_t sm = (size_t)(1 << (kWarpHashLog2 - 1)) * 8;
      set_smem(k_c4_block<NT8, true>, sm);
      int occ = 1;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_c4_block<NT8, true>, NT8, sm));
      const int g = std::min(cnt[7], c->sms * std::max(occ, 1));
      k_c4_block<NT8, true><<<g, NT8, sm, c->stream>>>(c->rp, c->ci, c->split, c->mir, lists[7], cnt[7],
                                                wc, parts, kWarpHashLog2 - 1, queues + 6, c4);
      check_launch();
      c->launched();
    }
    if (cnt[2] > 0) {  // class 3: 256-thread block-flattened tables of <= 4096 slots
      const size_t sm = (size_t)(1 << kC4SmallLog) * 8;
      set_smem(k_c4_block<256, true>, sm);
      int occ = 1;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_c4_block<256, true>, 256, sm));
      const int g = std::min(cnt[2], c->sms * std::max(occ, 1));
      k_c4_block<256, true><<<g, 256, sm, c->stream>>>(c->rp, c->ci, c->split, c->mir, lists[2], cnt[2],
                                                wc, parts, kC4SmallLog, queues + 0, c4);
      check_launch();
      c->launched();
    }
    if (cnt[3] > 0) {  // class 4: block-flattened hash-partition passes
      const size_t sm = (size_t)(1 << kC4HashLog) * 8;
      set_smem(k_c4_block<kC4BlockThreads>, sm);
      int occ = 1;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_c4_block<kC4BlockThreads>,
                                                       kC4BlockThreads, sm));
      const int g = std::min(cnt[3], c->sms * std::max(occ, 1));
      k_c4_block<kC4BlockThreads><<<g, kC4BlockThreads, sm, c->stream>>>(
          c->rp, c->ci, c->split, c->mir, lists[3], cnt[3], wc, parts, kC4HashLog, queues + 1, c4);
      check_launch();
      c->launched();
    }
    c->mark("c4 hash:end");
    c->mark("c4 dense:start");
    // classes 5/6 (big tiles) and 7 (small tiles): banded tile starts
    // (dense_span) and the absolute tile boundaries of the active rows
    const long long nact = (long long)c->nact;
    auto tiles_for = [&](long long tile_bytes, Buf tb_buf, Buf bnd_buf, int** bnd_out,
                         int* k_out) -> int* {
      std::vector<int> h{0};
      const long long t4 = 2 * tile_bytes, t8 = tile_bytes, t16 = tile_bytes / 2,
                      t32 = tile_bytes / 4;
      for (long long x = 0; x < nact;) {
        const long long e = x < bands[0] ? std::min<long long>(x + t4, bands[0])
                          : x < bands[1] ? std::min<long long>(x + t8, bands[1])
                          : x < bands[2] ? std::min<long long>(x + t16, bands[2])
                                         : std::min<long long>(x + t32, nact);
        h.push_back((int)e);
        x = e;
      }
      const long long K = (long long)h.size() - 1;
      *k_out = (int)K;
      int* tb = c->ensure<int>(tb_buf, h.size());
      CK(cudaMemcpyAsync(tb, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
      *bnd_out = nullptr;
      if (K * nact <= (1ll << 30)) {
        *bnd_out = c->ensure<int>(bnd_buf, (size_t)(K * nact));
        k_tile_bounds<<<c->grid(K * nact, 256), 256, 0, c->stream>>>(c->rp, c->ci, (int)nact,
                                                                      (int)K, tb, *bnd_out);
        check_launch();
        c->launched();
      }
      return tb;
    };
    if (cnt[4] > 0 || cnt[5] > 0) {
      int* bnd = nullptr;
      int K = 0;
      int* tb = tiles_for(kC4TileBytes, B_TB, B_TBND, &bnd, &K);
      for (int bb = 4; bb <= 5; ++bb) {
        if (cnt[bb] == 0) continue;
        const size_t sm = kC4TileBytes;
        // 32-bit-band roots (the few ranked above degree 65535) are huge: hand
        // out (root, tile) items so they spread over every SM
        const int skt = ((bb == 5 || FGLT_SPLIT_BIG) && bnd) ? K : 0;
        const int g = skt ? c->sms * (1024 / kC4DenseThreads)
                          : std::min(cnt[bb], c->sms * (1024 / kC4DenseThreads));
        int* cur = c->ensure<int>(B_CURSOR, 2 * (size_t)g * (size_t)(c->dmax + 1));
        if (bb == 4 && skt) {
          set_smem(k_c4_dense<true, kC4DenseThreads, true>, sm);
          k_c4_dense<true, kC4DenseThreads, true><<<g, kC4DenseThreads, sm, c->stream>>>(
              c->rp, c->ci, c->split, c->mir, lists[bb], cnt[bb], cur, (long long)(c->dmax + 1),
              bnd, nact, tb, bands[0], bands[1], bands[2], queues + 2, c4, skt);
        } else if (bb == 4) {
          set_smem(k_c4_dense<true, kC4DenseThreads>, sm);
          k_c4_dense<true, kC4DenseThreads><<<g, kC4DenseThreads, sm, c->stream>>>(
              c->rp, c->ci, c->split, c->mir, lists[bb], cnt[bb], cur, (long long)(c->dmax + 1),
              bnd, nact, tb, bands[0], bands[1], bands[2], queues + 2, c4, 0);
        } else {
          if (skt) {
            set_smem(k_c4_dense<false, kC4DenseThreads, true>, sm);
            k_c4_dense<false, kC4DenseThreads, true><<<g, kC4DenseThreads, sm, c->stream>>>(
                c->rp, c->ci, c->split, c->mir, lists[bb], cnt[bb], cur, (long long)(c->dmax + 1),
                bnd, nact, tb, bands[0], bands[1], bands[2], queues + 3, c4, skt);
          } else {
            set_smem(k_c4_dense<false, kC4DenseThreads>, sm);
            k_c4_dense<false, kC4DenseThreads><<<g, kC4DenseThreads, sm, c->stream>>>(
                c->rp, c->ci, c->split, c->mir, lists[bb], cnt[bb], cur, (long long)(c->dmax + 1),
                bnd, nact, tb, bands[0], bands[1], bands[2], queues + 3, c4, 0);
          }
        }
        check_launch();
        c->launched();
      }
    }
    if (cnt[6] > 0) {
      int* bnd = nullptr;
      int K = 0;
      int* tb = tiles_for(kC4TileBytesS, B_TBS, B_TBNDS, &bnd, &K);
      const size_t sm = kC4TileBytesS;
      const int g = std::min(cnt[6], c->sms * (1024 / kC4DenseThreadsS));
      int* cur = c->ensure<int>(B_CURSORS, 2 * (size_t)g * (size_t)(c->dmax + 1));
      set_smem(k_c4_dense<true, kC4DenseThreadsS>, sm);
      k_c4_dense<true, kC4DenseThreadsS><<<g, kC4DenseThreadsS, sm, c->stream>>>(
          c->rp, c->ci, c->split, c->mir, lists[6], cnt[6], cur, (long long)(c->dmax + 1), bnd,
          nact, tb, bands[0], bands[1], bands[2], queues + 5, c4, 0);
      check_launch();
      c->launched();
    }
    c->mark("c4 dense:end");
    c->mark("four-cycle rows:end");
  }
  if (P.d13) {
    root_bins(c, u0, u1);
    c->mark("roots:start");
    if (c->tl_u0 != u0 || c->tl_u1 != u1) c->tl = TriList{};  // list of another range
    c->mark("diamond list:start");
    diamond_list(c);
    c->mark("diamond list:end");
    c->mark("diamond probe:start");
    roots_pass<false, true, false>(c);
    c->mark("diamond probe:end");
    c->mark("roots:end");
  }
}

void epilogue(fglt_ctx* c, int64_t v0, int64_t v1, u64* raw, u64* net) {
  if (v1 <= v0) return;
  EpilogueIn in;
  in.rp = c->rp;
  in.inv = c->inv;
  const Plan& P = c->plan;
  in.p2 = P.p2 ? c->V(V_P2) : nullptr;
  in.p3 = P.p3 ? c->V(V_P3) : nullptr;
  in.c3 = P.c3 ? c->V(V_C3) : nullptr;
  in.d7 = P.d7 ? c->V(V_D7) : nullptr;
  in.d9 = P.d9 ? c->V(V_D9) : nullptr;
  in.d10 = P.d10 ? c->V(V_D10) : nullptr;
  in.d14 = P.d14 ? c->V(V_D14) : nullptr;
  in.c4 = P.c4 ? c->V(V_C4) : nullptr;
  in.d13 = P.d13 ? c->V(V_D13) : nullptr;
  in.d15 = P.d15 ? c->V(V_D15) : nullptr;
  const bool aligned =
      ((reinterpret_cast<uintptr_t>(raw) | reinterpret_cast<uintptr_t>(net)) & 15u) == 0;
  if (v0 == 0 && v1 == c->n && c->perm && c->inv)  // whole table: walk rows in vector order
    if (c->dict.mask == 0xFFFFu && aligned)
      k_epilogue_lines<<<c->grid(v1, kEpilogueThreads, 12), kEpilogueThreads, 0, c->stream>>>(
          in, c->perm, (int)v1, c->lenient, raw, net, c->d_small);
    else if (c->dict.mask == 0xFFFFu)
      k_epilogue_rank<true><<<c->grid(v1, kEpilogueThreads), kEpilogueThreads, 0, c->stream>>>(
          in, c->perm, c->d_dict, (int)v1, c->lenient, raw, net, c->d_small);
    else
      k_epilogue_rank<false><<<c->grid(v1, kEpilogueThreads), kEpilogueThreads, 0, c->stream>>>(
          in, c->perm, c->d_dict, (int)v1, c->lenient, raw, net, c->d_small);
  else
    k_epilogue<<<c->grid(v1 - v0, 128), 128, 0, c->stream>>>(in, c->d_dict, (int)v0, (int)v1,
                                                           c->lenient, raw, net, c->d_small);
  check_launch();
  c->launched();
}

// Decode the device error word into fglt_error; returns the code.
int read_error(fglt_ctx* c, fglt_error* err, bool sync = true) {
  u64 key = ~0ull;
  CK(cudaMemcpyAsync(&key, c->d_small, 8, cudaMemcpyDeviceToHost, c->stream));
  if (sync) CK(cudaStreamSynchronize(c->stream));
  if (err) err->order_key = key;
  if (key == ~0ull) return FGLT_OK;
  const int g = (int)(key & 15);
  const int code = (int)((key >> 4) & 15) ? FGLT_E_INCONSISTENCY : FGLT_E_OVERFLOW;
  const int64_t v = (int64_t)((key >> 8) & 0xffffffffull);
  if (code == FGLT_E_INCONSISTENCY)
    set_err(err, code, g, v,
            "negative net frequency for graphlet %d at vertex %lld (incomplete family or kernel defect)",
            g, (long long)v);
  else
    set_err(err, code, g, v, "count overflow (graphlet %d, vertex %lld)", g, (long long)v);
  if (err) err->order_key = key;
  return code;
}

void fill_stats(fglt_ctx* c, fglt_stats* st, const std::vector<std::pair<std::string, double>>& t) {
  if (!st) return;
  std::memset(st, 0, sizeof(*st));
  const Plan& P = c->plan;
  auto get = [&](const char* name) {
    double s = 0;
    for (auto& kv : t)
      if (kv.first == name) s += kv.second;
    return s;
  };
  // map measured phases onto the reference step names (see file header)
  double deg = get("degrees"), tri = get("triangles"), c4 = get("four-cycle rows"),
         rts = get("roots"), fill = get("column fill");
  bool ref_tri = false, ref_fc = false, ref_dia = false;
  for (auto& s : P.ref_steps) {
    ref_tri |= s == "triangles";
    ref_fc |= s == "four-cycle rows";
    ref_dia |= s == "diamond rows";
  }
  int k = 0;
  for (auto& s : P.ref_steps) {
    double v = 0;
    if (s == "degrees") v = deg;
    else if (s == "triangles") v = tri;
    else if (s == "four-cycle rows") v = c4 + (ref_tri ? 0 : tri);
    else if (s == "diamond rows") v = rts;
    else if (s == "tetrahedra") v = ref_dia ? 0 : rts;
    else if (s == "column fill") v = fill;
    if (k < FGLT_MAX_STEPS) {
      std::snprintf(st->step_names[k], 32, "%s", s.c_str());
      st->step_seconds[k] = v;
      ++k;
    }
  }
  (void)ref_fc;
  st->num_steps = k;
  if (!c->have_stats && c->n > 0) {
    read_graph_stats(c);
  }
  st->W = c->W;
  st->d_max = c->dmax;
  const bool four = (P.mask >> 12 & 1u) || (P.mask >> 14 & 1u);
  st->p2_row_touches = four ? c->W - 2 * (uint64_t)c->m : 0;
  st->p2_touch_bound = 2 * c->dmax * (uint64_t)c->m;
  st->peak_aux_words = c->peak_scratch / 8;
  st->largest_aux_alloc_words = c->largest / 8;
  st->threads_used = 1;
  st->device = c->device;
  st->kernel_launches = c->launches - c->launches_at_call;
  // every measured phase (reference steps and the finer device phases)
  std::vector<std::pair<std::string, u64>> units;
  if (!t.empty())
    for (auto& us : c->unit_slots) {
    u64 v = 0;
    CK(cudaMemcpy(&v, us.second, 8, cudaMemcpyDeviceToHost));
    units.push_back({us.first, v});
  }
  int np = 0;
  for (auto& kv : t) {
    if (np >= FGLT_MAX_PHASES) break;
    std::snprintf(st->phase_names[np], 32, "%s", kv.first.c_str());
    st->phase_seconds[np] = kv.second;
    st->phase_units[np] = 0;
    for (auto& u : units)
      if (u.first == kv.first) st->phase_units[np] = u.second;
    ++np;
  }
  st->num_phases = np;
}

std::vector<std::pair<std::string, double>> collect_marks(fglt_ctx* c) {
  std::vector<std::pair<std::string, double>> out;
  if (!c->timing || c->marks.empty()) return out;
  CK(cudaEventSynchronize(c->marks.back().second));
  for (size_t i = 0; i + 1 < c->marks.size(); ++i) {
    const std::string& a = c->marks[i].first;
    auto colon = a.find(':');
    if (colon == std::string::npos || a.substr(colon + 1) != "start") continue;
    const std::string name = a.substr(0, colon);
    for (size_t j = i + 1; j < c->marks.size(); ++j)
      if (c->marks[j].first == name + ":end") {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, c->marks[i].second, c->marks[j].second));
        out.push_back({name, ms * 1e-3});
        break;
      }
  }
  for (auto& mk : c->marks) cudaEventDestroy(mk.second);
  c->marks.clear();
  return out;
}

int validate_shape(int64_t n, int64_t nnz, fglt_error* err) {
  if (n < 0 || nnz < 0) {
    set_err(err, FGLT_E_STRUCTURAL, -1, -1, "negative graph size");
    return FGLT_E_STRUCTURAL;
  }
  if (n >= (int64_t)1 << 31 || nnz >= (int64_t)1 << 31) {
    set_err(err, FGLT_E_STRUCTURAL, -1, -1,
            "graph exceeds the int32 CSR limits (n=%lld, nnz=%lld)", (long long)n, (long long)nnz);
    return FGLT_E_STRUCTURAL;
  }
  if (nnz % 2) {
    set_err(err, FGLT_E_STRUCTURAL, -1, -1, "odd nnz: adjacency is not symmetric");
    return FGLT_E_STRUCTURAL;
  }
  return FGLT_OK;
}

}  // namespace

__global__ void __launch_bounds__(512, 2) k_probe_smem_atomics(int iters, unsigned words,
                                                                u64* __restrict__ sink) {
  extern __shared__ unsigned Lp[];
  for (unsigned i = threadIdx.x; i < words; i += blockDim.x) Lp[i] = 0;
  __syncthreads();
  unsigned x = blockIdx.x * blockDim.x + threadIdx.x + 1;
  for (int i = 0; i < iters; ++i) {
    x ^= x << 13;
    x ^= x >> 17;
    x ^= x << 5;
    atomicAdd(Lp + (x % words), 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) sink[blockIdx.x] = Lp[0];
}

// =================================================================== C-ABI
extern "C" {

uint64_t fglt_ctx_kernel_launches(const fglt_ctx* c) { return c ? c->launches : 0; }

int fglt_ctx_scratch_report(const fglt_ctx* c, char* out, int len) {
  if (!c || !out || len <= 0) return FGLT_E_NO_DEVICE;
  std::string r;
  for (int b = 0; b < B_COUNT; ++b)
    if (c->buf[b].p && c->buf[b].call == c->call)
      r += std::string(kBufName[b]) + " " + std::to_string(c->buf[b].req) +
           (is_staging(b) ? " staging\n" : "\n");
  std::snprintf(out, (size_t)len, "%s", r.c_str());
  return FGLT_OK;
}

int fglt_build_csr(fglt_ctx* c, const int64_t* eu, const int64_t* ev, int64_t ne,
                   int64_t declared_n, int symmetrize, int drop_self_loops, int dedupe,
                   uint32_t flags, int64_t* n_out, int64_t* nnz_out, int64_t* self_loops,
                   int64_t* duplicates, fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!c) {
    set_err(err, FGLT_E_NO_DEVICE, -1, -1, "null context");
    return FGLT_E_NO_DEVICE;
  }
  try {
    CK(cudaSetDevice(c->device));
    if (ne < 0 || declared_n < 0) {
      set_err(err, FGLT_E_STRUCTURAL, -1, -1, "negative size");
      return FGLT_E_STRUCTURAL;
    }
    if (2 * ne >= ((int64_t)1 << 31)) {
      set_err(err, FGLT_E_STRUCTURAL, -1, -1, "edge sample exceeds the int32 CSR limits");
      return FGLT_E_STRUCTURAL;
    }
    const bool mirror = symmetrize != 0;
    long long* de = c->ensure<long long>(B_ING_E, 2 * (size_t)std::max<int64_t>(ne, 1));
    const long long* du = reinterpret_cast<const long long*>(eu);
    const long long* dv = reinterpret_cast<const long long*>(ev);
    if (!(flags & FGLT_INPUT_DEVICE) && ne > 0) {
      CK(cudaMemcpyAsync(de, eu, (size_t)ne * 8, cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(de + ne, ev, (size_t)ne * 8, cudaMemcpyHostToDevice, c->stream));
      du = de;
      dv = de + ne;
    }
    c->d_small = c->ensure<u64>(B_SMALL, 64);
    CK(cudaMemsetAsync(c->d_small + 40, 0, 8 * sizeof(u64), c->stream));
    CK(cudaMemsetAsync(c->d_small + 43, 0xff, sizeof(u64), c->stream));
    u64 h[4] = {0, 0, 0, ~0ull};
    if (ne > 0) {
      k_ingest_scan<<<c->grid(ne, 256), 256, 0, c->stream>>>(du, dv, ne, c->d_small + 40);
      check_launch();
      c->launched();
      CK(cudaMemcpyAsync(h, c->d_small + 40, 32, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
    // error order and messages of build_adjacency (proj/src/graph.cpp:192-249)
    if (h[0]) {
      set_err(err, FGLT_E_STRUCTURAL, -1, -1, "negative vertex id in edge collection");
      return FGLT_E_STRUCTURAL;
    }
    if (h[1] && !drop_self_loops) {
      long long v = -1;
      CK(cudaMemcpyAsync(&v, du + h[3], 8, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      set_err(err, FGLT_E_STRUCTURAL, -1, (int64_t)v,
              "self-loop at vertex %lld (drop_self_loops is off)", v);
      return FGLT_E_STRUCTURAL;
    }
    const int64_t n = std::max<int64_t>(declared_n, ne > 0 ? (int64_t)h[2] + 1 : 0);
    if (n >= ((int64_t)1 << 31)) {
      set_err(err, FGLT_E_STRUCTURAL, -1, -1, "vertex ids exceed the int32 CSR limits");
      return FGLT_E_STRUCTURAL;
    }
    const int64_t nk = 2 * ne;
    u64* keys = c->ensure<u64>(B_ING_K, (size_t)std::max<int64_t>(nk, 1));
    u64* sorted = c->ensure<u64>(B_ING_K2, (size_t)std::max<int64_t>(nk, 1));
    int64_t nnz = 0;
    u64 dups = 0;
    if (ne > 0) {
      k_ingest_keys<<<c->grid(ne, 256), 256, 0, c->stream>>>(du, dv, ne, mirror ? 1 : 0, keys);
      check_launch();
      c->launched();
      int bits = 1;
      while (bits < 32 && ((int64_t)1 << bits) <= n) ++bits;
      size_t t1 = 0, t2 = 0;
      int* d_nsel = reinterpret_cast<int*>(c->d_small + 48);
      CK(cub::DeviceRadixSort::SortKeys(nullptr, t1, keys, sorted, (int)nk, 0, 64, c->stream));
      CK(cub::DeviceSelect::Unique(nullptr, t2, sorted, keys, d_nsel, (int)nk, c->stream));
      void* tmp = c->ensure<unsigned char>(B_CUB, std::max(t1, t2));
      size_t tb = c->buf[B_CUB].cap;
      // sentinels (~0) need the full 64 bits to sort last
      CK(cub::DeviceRadixSort::SortKeys(tmp, tb, keys, sorted, (int)nk, 0, 64, c->stream));
      c->launched();
      tb = c->buf[B_CUB].cap;
      CK(cub::DeviceSelect::Unique(tmp, tb, sorted, keys, d_nsel, (int)nk, c->stream));
      c->launched();
      int nsel = 0;
      u64 last = 0;
      CK(cudaMemcpyAsync(&nsel, d_nsel, 4, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if (nsel > 0)
        CK(cudaMemcpyAsync(&last, keys + nsel - 1, 8, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      nnz = nsel - (nsel > 0 && last == ~0ull ? 1 : 0);
      const int64_t valid = (mirror ? 2 : 1) * (ne - (int64_t)h[1]);
      dups = (u64)(valid - nnz);
      if (dups && !dedupe) {
        set_err(err, FGLT_E_STRUCTURAL, -1, -1, "duplicate edges present (dedupe is off)");
        return FGLT_E_STRUCTURAL;
      }
    }
    int* rp = c->ensure<int>(B_ING_RP, (size_t)n + 1);
    int* ci = c->ensure<int>(B_ING_CI, (size_t)std::max<int64_t>(nnz, 1));
    k_ingest_rows<<<c->grid(nnz + 1, 256), 256, 0, c->stream>>>(keys, nnz, (int)n, rp, ci);
    check_launch();
    c->launched();
    if (!mirror && nnz % 2) {
      set_err(err, FGLT_E_STRUCTURAL, -1, -1,
              "asymmetric input: odd number of directed entries with symmetrize off");
      return FGLT_E_STRUCTURAL;
    }
    if (!mirror && nnz > 0) {
      u64 init = ~0ull, bad = ~0ull;
      CK(cudaMemcpyAsync(c->d_small + 41, &init, 8, cudaMemcpyHostToDevice, c->stream));
      k_ingest_symmetric<<<c->grid(n, 256), 256, 0, c->stream>>>(rp, ci, (int)n, c->d_small + 41);
      check_launch();
      c->launched();
      CK(cudaMemcpyAsync(&bad, c->d_small + 41, 8, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if (bad != ~0ull) {
        set_err(err, FGLT_E_STRUCTURAL, -1, (int64_t)(bad >> 32),
                "asymmetric input: (%lld,%lld) present without its reverse and symmetrize off",
                (long long)(bad >> 32), (long long)(bad & 0xffffffffull));
        return FGLT_E_STRUCTURAL;
      }
    }
    CK(cudaStreamSynchronize(c->stream));
    c->ing_n = n;
    c->ing_nnz = nnz;
    if (n_out) *n_out = n;
    if (nnz_out) *nnz_out = nnz;
    if (self_loops) *self_loops = (int64_t)h[1];
    // undirected edges merged away: removed directed entries / 2 in both
    // modes, as the reference reports it (graph.cpp:227)
    if (duplicates) *duplicates = (int64_t)(dups / 2);
    return FGLT_OK;
  } catch (const CudaFail& f) {
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    return f.code;
  }
}

int fglt_csr_fetch(fglt_ctx* c, int32_t* row_ptr, int32_t* col_idx, uint32_t flags,
                   fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  try {
    CK(cudaSetDevice(c->device));
    const cudaMemcpyKind kind =
        (flags & FGLT_OUTPUT_DEVICE) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (row_ptr)
      CK(cudaMemcpyAsync(row_ptr, c->buf[B_ING_RP].p, (size_t)(c->ing_n + 1) * 4, kind, c->stream));
    if (col_idx && c->ing_nnz)
      CK(cudaMemcpyAsync(col_idx, c->buf[B_ING_CI].p, (size_t)c->ing_nnz * 4, kind, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return FGLT_OK;
  } catch (const CudaFail& f) {
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    return f.code;
  }
}

int fglt_ctx_set_debug(fglt_ctx* c, int key, int value) {
  if (!c) return FGLT_E_NO_DEVICE;
  switch (key) {
    case FGLT_DEBUG_C4_CLASS: c->force_c4_class = value; return FGLT_OK;
    case FGLT_DEBUG_C4_PARTS: c->force_c4_parts = value; return FGLT_OK;
    case FGLT_DEBUG_ROOTS_BIN: c->force_roots_bin = value; return FGLT_OK;
    case FGLT_DEBUG_HUB: c->force_hub = value; c->hub_built = false; return FGLT_OK;
    case FGLT_DEBUG_TRILIST: c->tl_mode = value; return FGLT_OK;
    case FGLT_DEBUG_ROW_SORT: c->force_row_sort = value; return FGLT_OK;
    case FGLT_DEBUG_FLAT_DMAX: c->flat_dmax = value < 0 ? 0 : value > 255 ? 255 : value; return FGLT_OK;
    default: return FGLT_E_PARSE;
  }
}

const char* fglt_version(void) { return "fglt-b200 0.2 (sm_100a)"; }

// Measured on-chip ceiling for the roofline of the dense 4-cycle kernel:
// random-address 32-bit shared-memory atomicAdd throughput with that
// kernel's tile size (96 KB) and occupancy (two 512-thread blocks per SM).
int fglt_probe_smem_atomics(fglt_ctx* c, double* ops_per_s, fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!c) return FGLT_E_NO_DEVICE;
  try {
    CK(cudaSetDevice(c->device));
    constexpr int kNT = 512, kIters = 4096;
    constexpr unsigned kWords = 98304 / 4;
    const int g = c->sms * 2;
    u64* sink = c->ensure<u64>(B_API5, (size_t)g);
    set_smem(k_probe_smem_atomics, kWords * 4);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_probe_smem_atomics<<<g, kNT, kWords * 4, c->stream>>>(kIters, kWords, sink);  // warm-up
    CK(cudaEventRecord(e0, c->stream));
    k_probe_smem_atomics<<<g, kNT, kWords * 4, c->stream>>>(kIters, kWords, sink);
    CK(cudaEventRecord(e1, c->stream));
    check_launch();
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ops_per_s = (double)g * kNT * kIters / (ms * 1e-3);
    return FGLT_OK;
  } catch (const CudaFail& f) {
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    return f.code;
  }
}

int fglt_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

fglt_ctx* fglt_ctx_create(int device, void* stream, fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    set_err(err, FGLT_E_NO_DEVICE, -1, -1, "no CUDA device available (%s); there is no CPU fallback",
            cudaGetErrorString(e));
    return nullptr;
  }
  if (device < 0 || device >= count) {
    set_err(err, FGLT_E_NO_DEVICE, -1, -1, "device %d out of range (%d devices)", device, count);
    return nullptr;
  }
  fglt_ctx* c = new fglt_ctx();
  try {
    c->device = device;
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) {
      set_err(err, FGLT_E_NO_DEVICE, -1, -1, "device %d is sm_%d%d; this build targets sm_100a",
              device, prop.major, prop.minor);
      delete c;
      return nullptr;
    }
    c->sms = prop.multiProcessorCount;
    c->stream = reinterpret_cast<cudaStream_t>(stream);
  } catch (const CudaFail& f) {
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    delete c;
    return nullptr;
  }
  return c;
}

int fglt_ctx_release_workspace(fglt_ctx* c) {
  if (!c) return FGLT_E_NO_DEVICE;
  if (cudaSetDevice(c->device) != cudaSuccess) return FGLT_E_CUDA;
  for (auto& b : c->buf) {
    if (b.p) cudaFreeAsync(b.p, c->stream);
    b.p = nullptr;
    b.cap = 0;
  }
  c->scratch_bytes = 0;
  c->n = c->nnz = c->m = 0;  // cached graph state refers to the freed buffers
  c->have_stats = false;
  c->rb_u0 = c->rb_u1 = -1;
  c->rb_cnt.clear();
  c->hub_built = false;
  c->big_rows_listed = false;
  c->tl = TriList{};
  c->tl_u0 = c->tl_u1 = -1;
  c->ing_n = c->ing_nnz = 0;
  return cudaStreamSynchronize(c->stream) == cudaSuccess ? FGLT_OK : FGLT_E_CUDA;
}

void fglt_ctx_destroy(fglt_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (auto& b : c->buf)
    if (b.p) cudaFreeAsync(b.p, c->stream);
  cudaStreamSynchronize(c->stream);
  delete c;
}

int fglt_ctx_transform(fglt_ctx* c, const int32_t* row_ptr, const int32_t* col_idx, int64_t n,
                       int64_t nnz, uint32_t dict_mask, int lenient, uint32_t flags,
                       uint64_t* raw_out, uint64_t* net_out, fglt_stats* stats,
                       fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!c) {
    set_err(err, FGLT_E_NO_DEVICE, -1, -1, "null context");
    return FGLT_E_NO_DEVICE;
  }
  if (dict_mask >> 16) {
    set_err(err, FGLT_E_PARSE, -1, -1, "graphlet id outside 0..15 in dictionary mask");
    return FGLT_E_PARSE;
  }
  int rc = validate_shape(n, nnz, err);
  if (rc) return rc;
  try {
    CK(cudaSetDevice(c->device));
    c->begin_call();
    c->timing = (flags & FGLT_TIMINGS) != 0;
    c->marks.clear();
    const int* d_rp = row_ptr;
    const int* d_ci = col_idx;
    c->mark("degrees:start");
    if (!(flags & FGLT_INPUT_DEVICE)) {
      int* a = c->ensure<int>(B_RP_IN, n + 1);
      int* b = c->ensure<int>(B_CI_IN, std::max<int64_t>(nnz, 1));
      CK(cudaMemcpyAsync(a, row_ptr, (size_t)(n + 1) * 4, cudaMemcpyHostToDevice, c->stream));
      if (nnz)
        CK(cudaMemcpyAsync(b, col_idx, (size_t)nnz * 4, cudaMemcpyHostToDevice, c->stream));
      d_rp = a;
      d_ci = b;
    }
    c->mark("prepare:start");
    prepare(c, d_rp, d_ci, n, nnz, dict_mask, lenient);
    if (c->plan.enumerate && !c->have_stats && n > 0) {
      // d_max sizes the 4-cycle cursor slices, max |N+(u)| the root bins
      read_graph_stats(c);
    }
    c->mark("prepare:end");
    c->mark("sweep A:start");
    sweep_a(c);
    c->mark("sweep A:end");
    c->mark("degrees:end");
    c->mark("triangles:start");
    triangles(c, 0, n);
    c->mark("sweeps B/C:start");
    local_sweeps(c);
    c->mark("sweeps B/C:end");
    c->mark("triangles:end");
    roots(c, 0, n);
    const size_t k = (size_t)c->dict.k;
    u64* raw = reinterpret_cast<u64*>(raw_out);
    u64* net = reinterpret_cast<u64*>(net_out);
    const bool dev_out = (flags & FGLT_OUTPUT_DEVICE) != 0;
    if (!dev_out) {
      raw = raw_out ? c->ensure<u64>(B_RAW, (size_t)std::max<int64_t>(n, 1) * k) : nullptr;
      net = net_out ? c->ensure<u64>(B_NET, (size_t)std::max<int64_t>(n, 1) * k) : nullptr;
    }
    c->mark("column fill:start");
    epilogue(c, 0, n, raw, net);
    c->mark("column fill:end");
    if (!dev_out && n > 0) {
      if (raw_out)
        CK(cudaMemcpyAsync(raw_out, raw, (size_t)n * k * 8, cudaMemcpyDeviceToHost, c->stream));
      if (net_out)
        CK(cudaMemcpyAsync(net_out, net, (size_t)n * k * 8, cudaMemcpyDeviceToHost, c->stream));
    }
    rc = read_error(c, err, true);
    auto t = collect_marks(c);
    // "roots" covers both diamond and tetrahedra phases
    fill_stats(c, stats, t);
    return rc;
  } catch (const CudaFail& f) {
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    return f.code;
  }
}

int fglt_transform_csr32(const int32_t* row_ptr, const int32_t* col_idx, int64_t n, int64_t nnz,
                         uint32_t dict_mask, int lenient, int device, uint32_t flags,
                         uint64_t* raw_out, uint64_t* net_out, fglt_stats* stats,
                         fglt_error* err) {
  fglt_ctx* c = fglt_ctx_create(device, nullptr, err);
  if (!c) return err ? err->code : FGLT_E_NO_DEVICE;
  int rc = fglt_ctx_transform(c, row_ptr, col_idx, n, nnz, dict_mask, lenient, flags, raw_out,
                              net_out, stats, err);
  fglt_ctx_destroy(c);
  return rc;
}

int fglt_net_from_raw(fglt_ctx* c, const uint64_t* raw, int64_t n, uint32_t dict_mask,
                      int lenient, uint64_t* net, fglt_error* err) {
  return fglt_net_from_raw_matrix(c, raw, n, dict_mask, nullptr, lenient, net, err);
}

int fglt_net_from_raw_matrix(fglt_ctx* c, const uint64_t* raw, int64_t n, uint32_t dict_mask,
                             const uint64_t* U, int lenient, uint64_t* net, fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!c) {
    set_err(err, FGLT_E_NO_DEVICE, -1, -1, "null context");
    return FGLT_E_NO_DEVICE;
  }
  try {
    CK(cudaSetDevice(c->device));
    c->begin_call();
    c->dict = make_dict(dict_mask);
    const size_t k = (size_t)c->dict.k;
    if (U) {  // the caller's unit upper-triangular matrix (ConversionMatrix, conversion.hpp:14-37)
      for (size_t r = 0; r < k; ++r)
        for (size_t col = 0; col <= r; ++col)
          if (U[r * k + col] != (col == r ? 1u : 0u)) {
            set_err(err, FGLT_E_STRUCTURAL, -1, -1,
                    "conversion matrix is not unit upper triangular at (%zu,%zu)", r, col);
            return FGLT_E_STRUCTURAL;
          }
      for (size_t r = 0; r < k; ++r) {
        int t = 0;
        for (size_t col = r + 1; col < k; ++col)
          if (U[r * k + col]) {
            c->dict.tail_col[r][t] = (int)col;
            c->dict.tail_coef[r][t] = U[r * k + col];
            ++t;
          }
        c->dict.ntail[r] = t;
      }
    }
    c->d_dict = c->ensure<DictInfo>(B_DICT, 1);
    CK(cudaMemcpyAsync(c->d_dict, &c->dict, sizeof(DictInfo), cudaMemcpyHostToDevice, c->stream));
    c->d_small = c->ensure<u64>(B_SMALL, 64);
    u64 init = ~0ull;
    CK(cudaMemcpyAsync(c->d_small, &init, 8, cudaMemcpyHostToDevice, c->stream));
    if (n > 0) {
      u64* dr = c->ensure<u64>(B_RAW, (size_t)n * k);
      u64* dn = c->ensure<u64>(B_NET, (size_t)n * k);
      CK(cudaMemcpyAsync(dr, raw, (size_t)n * k * 8, cudaMemcpyHostToDevice, c->stream));
      k_net_only<<<c->grid(n, 128), 128, 0, c->stream>>>(dr, c->d_dict, n, lenient, dn, c->d_small);
      check_launch();
      c->launched();
      CK(cudaMemcpyAsync(net, dn, (size_t)n * k * 8, cudaMemcpyDeviceToHost, c->stream));
    }
    return read_error(c, err, true);
  } catch (const CudaFail& f) {
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    return f.code;
  }
}

// ------------------------------------------------------------------ staged
int fglt_stage_prepare(fglt_ctx* c, const int32_t* d_row_ptr, const int32_t* d_col_idx, int64_t n,
                       int64_t nnz, uint32_t dict_mask, int lenient, fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  int rc = validate_shape(n, nnz, err);
  if (rc) return rc;
  try {
    CK(cudaSetDevice(c->device));
    c->begin_call();
    c->timing = false;
    prepare(c, d_row_ptr, d_col_idx, n, nnz, dict_mask, lenient);
    if (n > 0) {
      read_graph_stats(c);
    }
    sweep_a(c);
    return FGLT_OK;
  } catch (const CudaFail& f) {
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    return f.code;
  }
}

// Contiguous root blocks of (nearly) equal exact work: per root u,
// work(u) = wedges(u) + triangle probes(u) + 1, prefix-summed on the device;
// rank r's block starts at the first root whose inclusive prefix reaches
// total * r / world.
__global__ void k_work_total(const u64* __restrict__ wc, const u64* __restrict__ tw, int n,
                             u64* __restrict__ out) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x)
    out[u] = wc[u] + tw[u] + 1;
}

__global__ void k_cut_bounds(const u64* __restrict__ pre, int n, int world,
                             long long* __restrict__ bounds) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > world) return;
  if (r == 0 || r == world) {
    bounds[r] = r == 0 ? 0 : n;
    return;
  }
  const u64 total = pre[n - 1];
  const u64 target = (u64)(((unsigned __int128)total * (unsigned)r) / (unsigned)world);
  int lo = 0, hi = n;  // first u with pre[u] >= target; the block starts after it
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (pre[mid] < target) lo = mid + 1; else hi = mid;
  }
  bounds[r] = lo < n ? lo + 1 : n;
}

int fglt_stage_bounds(fglt_ctx* c, int world, int64_t* bounds, fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  try {
    CK(cudaSetDevice(c->device));
    const int64_t n = c->n;
    bounds[0] = 0;
    for (int r = 1; r <= world; ++r) bounds[r] = n;
    if (n == 0 || world <= 1 || !c->plan.enumerate) {
      for (int r = 1; r < world; ++r) bounds[r] = n * r / world;
      return FGLT_OK;
    }
    u64* work = c->ensure<u64>(B_WORK, 3 * (size_t)n);
    const int G = group_for((double)c->nnz / (double)n);
    DISPATCH_G(G, launch_root_work, c, work);
    DISPATCH_G(G, launch_probe_work, c, work + n);
    k_work_total<<<c->grid(n, 256), 256, 0, c->stream>>>(work, work + n, (int)n, work + 2 * n);
    check_launch();
    c->launched();
    size_t tb = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tb, work + 2 * n, work, (int)n, c->stream));
    void* tmp = c->ensure<unsigned char>(B_CUB, tb);
    CK(cub::DeviceScan::InclusiveSum(tmp, tb, work + 2 * n, work, (int)n, c->stream));
    c->launched();
    long long* d_b = c->ensure<long long>(B_API0, (size_t)world + 1);
    k_cut_bounds<<<(world + 128) / 128, 128, 0, c->stream>>>(work, (int)n, world, d_b);
    check_launch();
    c->launched();
    CK(cudaMemcpyAsync(bounds, d_b, ((size_t)world + 1) * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int r = 1; r <= world; ++r) bounds[r] = std::max(bounds[r], bounds[r - 1]);
    return FGLT_OK;
  } catch (const CudaFail& f) {
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    return f.code;
  }
}

int fglt_stage_triangles(fglt_ctx* c, int64_t u0, int64_t u1, uint32_t** d_edge_counts,
                         int64_t* count, fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  try {
    CK(cudaSetDevice(c->device));
    *d_edge_counts = c->C3f;
    *count = c->plan.c3 ? c->nnz : 0;
    triangles(c, u0, u1);
    CK(cudaStreamSynchronize(c->stream));
    return FGLT_OK;
  } catch (const CudaFail& f) {
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    return f.code;
  }
}

int fglt_stage_local(fglt_ctx* c, fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  try {
    CK(cudaSetDevice(c->device));
    local_sweeps(c);
    return FGLT_OK;
  } catch (const CudaFail& f) {
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    return f.code;
  }
}

// Row-partitioned vertex sweeps of rank `part` of `nparts` (rows r = part mod
// nparts). phase 0: sweep B (c3, d14, d10, p3 of my rows; the other rows stay
// 0) and *d_c3 / *count = the c3 vector to sum over ranks before phase 1;
// phase 1: sweep C (d9 of my rows, reads every row's c3). fglt_stage_roots
// then hands out d14..d15 (7 n values) instead of c4..d15 for the final sum.
int fglt_stage_local_part(fglt_ctx* c, int part, int nparts, int phase, uint64_t** d_c3,
                          int64_t* count, fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (nparts < 1 || part < 0 || part >= nparts || (phase != 0 && phase != 1)) {
    set_err(err, FGLT_E_PARSE, -1, -1, "fglt_stage_local_part: bad part / phase");
    return FGLT_E_PARSE;
  }
  try {
    CK(cudaSetDevice(c->device));
    c->rows_part = part;
    c->rows_parts = nparts;
    c->local_partial = nparts > 1;
    local_sweeps(c, false, phase == 0 ? 1 : 2);
    c->rows_part = 0;
    c->rows_parts = 1;
    if (d_c3) *d_c3 = reinterpret_cast<uint64_t*>(c->V(V_C3));
    if (count) *count = (phase == 0 && c->plan.c3 && nparts > 1) ? c->n : 0;
    if (phase == 0) CK(cudaStreamSynchronize(c->stream));
    return FGLT_OK;
  } catch (const CudaFail& f) {
    c->rows_part = 0;
    c->rows_parts = 1;
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    return f.code;
  }
}

int fglt_stage_roots(fglt_ctx* c, int64_t u0, int64_t u1, uint64_t** d_vectors, int64_t* count,
                     fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  try {
    CK(cudaSetDevice(c->device));
    roots(c, u0, u1);
    CK(cudaStreamSynchronize(c->stream));
    // d14, d10, p3, d9, c4, d13, d15 are contiguous in B_VEC; after
    // row-partitioned sweeps the first four are partial too
    *d_vectors = reinterpret_cast<uint64_t*>(c->V(c->local_partial ? V_D14 : V_C4));
    *count = (c->local_partial ? 7 : 3) * c->n;
    return FGLT_OK;
  } catch (const CudaFail& f) {
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    return f.code;
  }
}

int fglt_stage_epilogue(fglt_ctx* c, int64_t v0, int64_t v1, uint64_t* d_raw_rows,
                        uint64_t* d_net_rows, fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  try {
    CK(cudaSetDevice(c->device));
    epilogue(c, v0, v1, reinterpret_cast<u64*>(d_raw_rows), reinterpret_cast<u64*>(d_net_rows));
    return read_error(c, err, true);
  } catch (const CudaFail& f) {
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    return f.code;
  }
}

}  // extern "C"

// ------------------------------------------------------------- per-kernel
// The reference's public per-kernel functions (kernels.hpp:43-98) on the
// device; host arrays in and out (fglt_kernels_api.cuh).
namespace {

struct ApiCall {
  fglt_ctx* c;
  fglt_error* err;
  const int* d_rp = nullptr;
  const int* d_ci = nullptr;
};

// Device copies of the CSR (when given) and a fresh error word.
void api_begin(ApiCall& a, const int32_t* rp, const int32_t* ci, int64_t n, int64_t nnz) {
  fglt_ctx* c = a.c;
  CK(cudaSetDevice(c->device));
  c->begin_call();
  c->timing = false;
  c->d_small = c->ensure<u64>(B_SMALL, 64);
  u64 init = ~0ull;
  CK(cudaMemcpyAsync(c->d_small, &init, 8, cudaMemcpyHostToDevice, c->stream));
  if (rp) {
    int* drp = c->ensure<int>(B_RP_IN, n + 1);
    int* dci = c->ensure<int>(B_CI_IN, std::max<int64_t>(nnz, 1));
    CK(cudaMemcpyAsync(drp, rp, (size_t)(n + 1) * 4, cudaMemcpyHostToDevice, c->stream));
    if (nnz) CK(cudaMemcpyAsync(dci, ci, (size_t)nnz * 4, cudaMemcpyHostToDevice, c->stream));
    a.d_rp = drp;
    a.d_ci = dci;
  }
}

u64* api_upload(fglt_ctx* c, Buf b, const uint64_t* h, int64_t cnt) {
  u64* d = c->ensure<u64>(b, (size_t)std::max<int64_t>(cnt, 1));
  if (cnt > 0) CK(cudaMemcpyAsync(d, h, (size_t)cnt * 8, cudaMemcpyHostToDevice, c->stream));
  return d;
}

void api_download(fglt_ctx* c, uint64_t* h, const u64* d, int64_t cnt) {
  if (cnt > 0 && h) CK(cudaMemcpyAsync(h, d, (size_t)cnt * 8, cudaMemcpyDeviceToHost, c->stream));
}

template <class F>
int api_run(fglt_ctx* c, fglt_error* err, int64_t n, int64_t nnz, bool csr, F&& body) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!c) {
    set_err(err, FGLT_E_NO_DEVICE, -1, -1, "null context");
    return FGLT_E_NO_DEVICE;
  }
  int rc = csr ? validate_shape(n, nnz, err) : (n < 0 || n >= ((int64_t)1 << 31) ? FGLT_E_STRUCTURAL : 0);
  if (rc) {
    if (!csr) set_err(err, rc, -1, -1, "vector length outside the int32 limits");
    return rc;
  }
  try {
    body();
    return read_error(c, err, true);
  } catch (const CudaFail& f) {
    set_err(err, f.code, -1, -1, "%s", f.msg.c_str());
    return f.code;
  }
}

// Relabelled pipeline up to the per-edge triangle counts (and optionally the
// diamond roots); C3/c3 land in original order in B_API4 / B_API5.
void api_c3(fglt_ctx* c, const int* d_rp, const int* d_ci, int64_t n, int64_t nnz, bool d13) {
  const unsigned mask = 3u | (1u << 4) | (d13 ? (1u << 13) : 0u);
  prepare(c, d_rp, d_ci, n, nnz, mask, 1);
  u64* C3 = c->ensure<u64>(B_API4, (size_t)std::max<int64_t>(nnz, 1));
  u64* c3 = c->ensure<u64>(B_API5, (size_t)std::max<int64_t>(n, 1));
  if (n == 0) return;
  read_graph_stats(c);
  triangles(c, 0, n);
  local_sweeps(c, true);
  k_api_map_c3<<<c->grid(n * 32, 256), 256, 0, c->stream>>>(d_rp, d_ci, (int)n, c->inv, c->rp,
                                                           c->ci, c->C3f, c->V(V_C3), C3, c3);
  check_launch();
  c->launched();
}

}  // namespace

extern "C" {

int fglt_kernel_p2(fglt_ctx* c, const int32_t* rp, const int32_t* ci, int64_t n, int64_t nnz,
                   const uint64_t* p1, uint64_t* p2, fglt_error* err) {
  return api_run(c, err, n, nnz, true, [&] {
    ApiCall a{c, err};
    api_begin(a, rp, ci, n, nnz);
    u64* dp1 = api_upload(c, B_API0, p1, n);
    u64* out = c->ensure<u64>(B_API1, (size_t)std::max<int64_t>(n, 1));
    if (n) {
      k_api_p2<<<c->grid(n, 128), 128, 0, c->stream>>>(a.d_rp, a.d_ci, (int)n, dp1, out);
      check_launch();
      c->launched();
    }
    api_download(c, p2, out, n);
  });
}

int fglt_kernel_p3(fglt_ctx* c, const int32_t* rp, const int32_t* ci, int64_t n, int64_t nnz,
                   const uint64_t* p1, const uint64_t* p2, const uint64_t* c3, uint64_t* p3,
                   fglt_error* err) {
  return api_run(c, err, n, nnz, true, [&] {
    ApiCall a{c, err};
    api_begin(a, rp, ci, n, nnz);
    u64* dp1 = api_upload(c, B_API0, p1, n);
    u64* dp2 = api_upload(c, B_API1, p2, n);
    u64* dc3 = api_upload(c, B_API2, c3, n);
    u64* out = c->ensure<u64>(B_API3, (size_t)std::max<int64_t>(n, 1));
    if (n) {
      k_api_p3<<<c->grid(n, 128), 128, 0, c->stream>>>(a.d_rp, a.d_ci, (int)n, dp1, dp2, dc3, out);
      check_launch();
      c->launched();
    }
    api_download(c, p3, out, n);
  });
}

int fglt_kernel_d7(fglt_ctx* c, const int32_t* rp, const int32_t* ci, int64_t n, int64_t nnz,
                   const uint64_t* p1, uint64_t* d7, fglt_error* err) {
  return api_run(c, err, n, nnz, true, [&] {
    ApiCall a{c, err};
    api_begin(a, rp, ci, n, nnz);
    u64* dp1 = api_upload(c, B_API0, p1, n);
    u64* out = c->ensure<u64>(B_API1, (size_t)std::max<int64_t>(n, 1));
    if (n) {
      k_api_d7<<<c->grid(n, 128), 128, 0, c->stream>>>(a.d_rp, a.d_ci, (int)n, dp1, out, c->d_small);
      check_launch();
      c->launched();
    }
    api_download(c, d7, out, n);
  });
}

int fglt_kernel_d8(fglt_ctx* c, int64_t n, const uint64_t* p1, uint64_t* d8, fglt_error* err) {
  return api_run(c, err, n, 0, false, [&] {
    ApiCall a{c, err};
    api_begin(a, nullptr, nullptr, n, 0);
    u64* dp1 = api_upload(c, B_API0, p1, n);
    u64* out = c->ensure<u64>(B_API1, (size_t)std::max<int64_t>(n, 1));
    if (n) {
      k_api_d8<<<c->grid(n, 128), 128, 0, c->stream>>>((int)n, dp1, out, c->d_small);
      check_launch();
      c->launched();
    }
    api_download(c, d8, out, n);
  });
}

int fglt_kernel_d9_d10_d11(fglt_ctx* c, const int32_t* rp, const int32_t* ci, int64_t n,
                           int64_t nnz, const uint64_t* p1, const uint64_t* c3,
                           const uint64_t* C3, uint64_t* d9, uint64_t* d10, uint64_t* d11,
                           fglt_error* err) {
  return api_run(c, err, n, nnz, true, [&] {
    ApiCall a{c, err};
    api_begin(a, rp, ci, n, nnz);
    u64* dp1 = api_upload(c, B_API0, p1, n);
    u64* dc3 = api_upload(c, B_API1, c3, n);
    u64* dC3 = api_upload(c, B_API2, C3, nnz);
    u64* out = c->ensure<u64>(B_API3, 3 * (size_t)std::max<int64_t>(n, 1));
    if (n) {
      k_api_d9_11<<<c->grid(n, 128), 128, 0, c->stream>>>(a.d_rp, a.d_ci, (int)n, dp1, dc3, dC3,
                                                         out, out + n, out + 2 * n, c->d_small);
      check_launch();
      c->launched();
    }
    api_download(c, d9, out, n);
    api_download(c, d10, out + n, n);
    api_download(c, d11, out + 2 * n, n);
  });
}

int fglt_kernel_c3(fglt_ctx* c, const int32_t* rp, const int32_t* ci, int64_t n, int64_t nnz,
                   uint64_t* c3, uint64_t* C3, fglt_error* err) {
  return api_run(c, err, n, nnz, true, [&] {
    ApiCall a{c, err};
    api_begin(a, rp, ci, n, nnz);
    api_c3(c, a.d_rp, a.d_ci, n, nnz, false);
    api_download(c, C3, reinterpret_cast<u64*>(c->buf[B_API4].p), nnz);
    api_download(c, c3, reinterpret_cast<u64*>(c->buf[B_API5].p), n);
  });
}

int fglt_kernel_d13(fglt_ctx* c, const int32_t* rp, const int32_t* ci, int64_t n, int64_t nnz,
                    const uint64_t* C3, uint64_t* d13, fglt_error* err) {
  return api_run(c, err, n, nnz, true, [&] {
    ApiCall a{c, err};
    api_begin(a, rp, ci, n, nnz);
    u64* given = api_upload(c, B_API0, C3, nnz);
    u64* out = c->ensure<u64>(B_API1, (size_t)std::max<int64_t>(n, 1));
    if (n == 0) return;
    // The caller's C3 is usually the graph's own (compute_c3_C3): then the
    // root-centric diamond pass applies. Any other C3 is honoured literally.
    api_c3(c, a.d_rp, a.d_ci, n, nnz, true);
    unsigned long long* nd = reinterpret_cast<unsigned long long*>(c->d_small + 40);
    CK(cudaMemsetAsync(nd, 0, 8, c->stream));
    if (nnz) {
      k_api_diff<<<c->grid(nnz, 256), 256, 0, c->stream>>>(
          given, reinterpret_cast<u64*>(c->buf[B_API4].p), nnz, nd);
      check_launch();
      c->launched();
    }
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, nd, 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (h == 0) {
      roots(c, 0, n);
      k_api_gather<<<c->grid(n, 256), 256, 0, c->stream>>>(c->V(V_D13), c->inv, (int)n, out);
    } else {
      k_api_d13<<<c->grid(n * 32, 256), 256, 0, c->stream>>>(a.d_rp, a.d_ci, (int)n, given, out);
    }
    check_launch();
    c->launched();
    api_download(c, d13, out, n);
  });
}

}  // extern "C"
