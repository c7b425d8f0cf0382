// fglt_multi.cpp — single-process multi-GPU transform behind the C-ABI
// (include/fglt.h fglt_transform_multi): one host thread and
// one fglt_ctx per device, NCCL communicators from ncclCommInitAll, the
// staged pipeline of fglt.cu per rank:
//
//   broadcast CSR from devices[0] (ncclBroadcast over NVLink)
//   stage_prepare (replicated: degree relabel + split/mirror)
//   stage_bounds  (contiguous root blocks of equal exact work)
//   stage_triangles(own roots) -> ncclAllReduce(sum) of the uint32 per-edge C3
//   stage_local_part(rows r = rank mod world): sweep B -> ncclAllReduce(sum) of
//                 the n uint64 c3 -> sweep C
//   stage_roots(own roots)     -> ncclAllReduce(sum) of the 7n uint64
//                 d14/d10/p3/d9 (my rows) + c4/d13/d15 (my roots)
//   stage_epilogue(own block of ORIGINAL ids) -> rows straight to the caller's
//                  tables (D2H, or a peer copy to devices[0])
//
// Integer sums are associative, so the tables are byte-identical for any
// device count (tests/test_multi_device.py). A device list with repeats (e.g.
// {0, 0}) cannot form an NCCL clique; it runs the same ranks one after the
// other on that device with host-staged sums instead — the correctness path
// for more ranks than GPUs (no rank ever waits on another rank's kernel).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is opened at run time (see Nccl)

#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fglt.h"

namespace {

struct Fail {
  int code;
  std::string msg;
};

#define MCK(call)                                                                       \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) throw Fail{FGLT_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)
// NCCL is opened on first multi-GPU use instead of being linked: a process
// that also loads PyTorch must keep ONE libnccl.so.2 (torch bundles its own,
// newer than the system copy), so an already-loaded libnccl is reused
// (RTLD_NOLOAD) and the system library is opened only when none is loaded.
struct Nccl {
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = std::getenv("FGLT_NCCL_LIB");
    void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(dlsym(h, "ncclBroadcast"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
    api.GetErrorString =
        reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!api.CommInitAll || !api.Broadcast || !api.AllReduce || !api.GetErrorString)
    throw Fail{FGLT_E_CUDA, "libnccl.so.2 could not be loaded (set FGLT_NCCL_LIB)"};
  return api;
}

#define NCK(call)                                                                       \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      throw Fail{FGLT_E_CUDA, std::string(#call) + ": " + nccl().GetErrorString(r_)};  \
  } while (0)

void put(fglt_error* err, int code, const std::string& msg) {
  if (!err) return;
  err->code = code;
  err->graphlet_id = -1;
  err->vertex = -1;
  std::snprintf(err->msg, sizeof(err->msg), "%s", msg.c_str());
}

// Device buffer that grows (never shrinks) between calls.
struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  int dev = 0;
  void* get(size_t bytes) {
    if (cap < bytes) {
      if (p) cudaFree(p);
      p = nullptr;
      MCK(cudaSetDevice(dev));
      MCK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
      cap = std::max<size_t>(bytes, 16);
    }
    return p;
  }
  ~DBuf() {
    if (p) {
      cudaSetDevice(dev);
      cudaFree(p);
    }
  }
};

struct Rank {
  int dev = 0;
  cudaStream_t stream = nullptr;
  fglt_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  DBuf rp, ci, raw, net;
};

// One cached group per device list (contexts, streams, communicators).
struct Group {
  std::vector<int> devices;
  bool emulated = false;  // repeated devices: host-staged collectives, ranks in sequence
  std::vector<std::unique_ptr<Rank>> ranks;
  std::mutex run;

  ~Group() {
    for (auto& r : ranks) {
      cudaSetDevice(r->dev);
      if (r->comm && nccl().CommDestroy) nccl().CommDestroy(r->comm);
      if (r->ctx) fglt_ctx_destroy(r->ctx);
      if (r->stream) cudaStreamDestroy(r->stream);
    }
  }
};

std::mutex g_groups_mu;
std::map<std::vector<int>, std::unique_ptr<Group>> g_groups;

Group* group_for(const int* devices, int num) {
  std::vector<int> key(devices, devices + num);
  std::lock_guard<std::mutex> lock(g_groups_mu);
  auto it = g_groups.find(key);
  if (it != g_groups.end()) return it->second.get();
  auto g = std::make_unique<Group>();
  g->devices = key;
  std::vector<int> sorted = key;
  std::sort(sorted.begin(), sorted.end());
  g->emulated = std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end();
  for (int d : key) {
    auto r = std::make_unique<Rank>();
    r->dev = d;
    r->rp.dev = r->ci.dev = r->raw.dev = r->net.dev = d;
    MCK(cudaSetDevice(d));
    MCK(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
    fglt_error e{};
    r->ctx = fglt_ctx_create(d, r->stream, &e);
    if (!r->ctx) throw Fail{e.code ? e.code : FGLT_E_NO_DEVICE, e.msg};
    g->ranks.push_back(std::move(r));
  }
  if (!g->emulated && num > 1) {
    std::vector<ncclComm_t> comms((size_t)num);
    NCK(nccl().CommInitAll(comms.data(), num, key.data()));
    for (int i = 0; i < num; ++i) g->ranks[(size_t)i]->comm = comms[(size_t)i];
  }
  Group* raw = g.get();
  g_groups[key] = std::move(g);
  return raw;
}

// Per-rank outcome of the staged pipeline.
struct Outcome {
  int rc = FGLT_OK;
  fglt_error err{};
  fglt_stats st{};
};

void stage_check(int rc, const fglt_error& e, Outcome* o) {
  if (rc) {
    o->rc = rc;
    o->err = e;
    throw Fail{rc, e.msg};
  }
}

struct Job {
  const int32_t* rp;
  const int32_t* ci;
  int64_t n, nnz;
  uint32_t mask;
  int lenient;
  uint32_t flags;
  uint64_t* raw_out;
  uint64_t* net_out;
  int k;
  std::vector<int64_t> blocks;  // original-id row blocks, world + 1 entries
};

// Steps 1-2 of a rank: CSR on the device (copy or broadcast), prepare, bounds.
void rank_prepare(Group* g, int r, const Job& j, std::vector<int64_t>* bounds, Outcome* o) {
  Rank& R = *g->ranks[(size_t)r];
  const int world = (int)g->ranks.size();
  MCK(cudaSetDevice(R.dev));
  auto* drp = static_cast<int32_t*>(R.rp.get((size_t)(j.n + 1) * 4));
  auto* dci = static_cast<int32_t*>(R.ci.get((size_t)std::max<int64_t>(j.nnz, 1) * 4));
  const bool dev_in = (j.flags & FGLT_INPUT_DEVICE) != 0;
  if (g->emulated || world == 1) {
    const cudaMemcpyKind kind = dev_in ? cudaMemcpyDefault : cudaMemcpyHostToDevice;
    MCK(cudaMemcpyAsync(drp, j.rp, (size_t)(j.n + 1) * 4, kind, R.stream));
    if (j.nnz) MCK(cudaMemcpyAsync(dci, j.ci, (size_t)j.nnz * 4, kind, R.stream));
  } else {
    if (r == 0) {  // devices[0] holds (or receives) the input
      const cudaMemcpyKind kind = dev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
      MCK(cudaMemcpyAsync(drp, j.rp, (size_t)(j.n + 1) * 4, kind, R.stream));
      if (j.nnz) MCK(cudaMemcpyAsync(dci, j.ci, (size_t)j.nnz * 4, kind, R.stream));
    }
    NCK(nccl().Broadcast(drp, drp, (size_t)(j.n + 1), ncclInt32, 0, R.comm, R.stream));
    if (j.nnz) NCK(nccl().Broadcast(dci, dci, (size_t)j.nnz, ncclInt32, 0, R.comm, R.stream));
  }
  fglt_error e{};
  stage_check(fglt_stage_prepare(R.ctx, drp, j.nnz ? dci : nullptr, j.n, j.nnz, j.mask, j.lenient,
                                 &e), e, o);
  bounds->assign((size_t)world + 1, 0);
  stage_check(fglt_stage_bounds(R.ctx, world, bounds->data(), &e), e, o);
}

void rank_epilogue(Group* g, int r, const Job& j, Outcome* o) {
  Rank& R = *g->ranks[(size_t)r];
  MCK(cudaSetDevice(R.dev));
  const int64_t v0 = j.blocks[(size_t)r], v1 = j.blocks[(size_t)r + 1];
  const size_t rows = (size_t)std::max<int64_t>(v1 - v0, 0);
  auto* draw = j.raw_out ? static_cast<uint64_t*>(R.raw.get(rows * j.k * 8)) : nullptr;
  auto* dnet = j.net_out ? static_cast<uint64_t*>(R.net.get(rows * j.k * 8)) : nullptr;
  fglt_error e{};
  const int rc = fglt_stage_epilogue(R.ctx, v0, v1, draw, dnet, &e);
  if (rc) {  // combined across ranks by order key (first failure in reference order)
    o->rc = rc;
    o->err = e;
    return;
  }
  if (!rows) return;
  const bool dev_out = (j.flags & FGLT_OUTPUT_DEVICE) != 0;
  const size_t off = (size_t)v0 * j.k, bytes = rows * j.k * 8;
  if (draw) MCK(cudaMemcpyAsync(j.raw_out + off, draw, bytes, dev_out ? cudaMemcpyDefault : cudaMemcpyDeviceToHost, R.stream));
  if (dnet) MCK(cudaMemcpyAsync(j.net_out + off, dnet, bytes, dev_out ? cudaMemcpyDefault : cudaMemcpyDeviceToHost, R.stream));
  MCK(cudaStreamSynchronize(R.stream));
}

// Real multi-GPU rank: runs concurrently with the others, NCCL collectives.
void rank_nccl(Group* g, int r, const Job* jp, Outcome* o) {
  try {
    Rank& R = *g->ranks[(size_t)r];
    Job j = *jp;
    std::vector<int64_t> b;
    rank_prepare(g, r, j, &b, o);
    const int64_t u0 = b[(size_t)r], u1 = b[(size_t)r + 1];
    fglt_error e{};
    uint32_t* c3 = nullptr;
    int64_t cnt = 0;
    stage_check(fglt_stage_triangles(R.ctx, u0, u1, &c3, &cnt, &e), e, o);
    if (cnt && g->ranks.size() > 1)
      NCK(nccl().AllReduce(c3, c3, (size_t)cnt, ncclUint32, ncclSum, R.comm, R.stream));
    // vertex sweeps on my rows (r = rank mod world); sweep C reads every
    // row's c3, so that vector is summed in between
    const int world = (int)g->ranks.size();
    uint64_t* c3v = nullptr;
    stage_check(fglt_stage_local_part(R.ctx, r, world, 0, &c3v, &cnt, &e), e, o);
    if (cnt && world > 1)
      NCK(nccl().AllReduce(c3v, c3v, (size_t)cnt, ncclUint64, ncclSum, R.comm, R.stream));
    stage_check(fglt_stage_local_part(R.ctx, r, world, 1, nullptr, nullptr, &e), e, o);
    uint64_t* vec = nullptr;
    stage_check(fglt_stage_roots(R.ctx, u0, u1, &vec, &cnt, &e), e, o);
    if (cnt && world > 1)
      NCK(nccl().AllReduce(vec, vec, (size_t)cnt, ncclUint64, ncclSum, R.comm, R.stream));
    rank_epilogue(g, r, j, o);
  } catch (const Fail& f) {
    if (!o->rc) {
      o->rc = f.code;
      put(&o->err, f.code, f.msg);
    }
  }
}

// Ranks sharing devices: same stages in sequence, sums staged through the host.
void run_emulated(Group* g, const Job& j, std::vector<Outcome>* outs) {
  const int world = (int)g->ranks.size();
  std::vector<std::vector<int64_t>> b((size_t)world);
  for (int r = 0; r < world; ++r) rank_prepare(g, r, j, &b[(size_t)r], &(*outs)[(size_t)r]);
  auto host_sum = [&](std::vector<void*>& ptrs, int64_t cnt, size_t elem) {
    std::vector<uint64_t> acc((size_t)cnt, 0), part((size_t)cnt);
    for (int r = 0; r < world; ++r) {
      Rank& R = *g->ranks[(size_t)r];
      MCK(cudaSetDevice(R.dev));
      MCK(cudaMemcpyAsync(part.data(), ptrs[(size_t)r], (size_t)cnt * elem, cudaMemcpyDeviceToHost, R.stream));
      MCK(cudaStreamSynchronize(R.stream));
      if (elem == 4) {
        const uint32_t* p = reinterpret_cast<const uint32_t*>(part.data());
        auto* a = reinterpret_cast<uint32_t*>(acc.data());
        for (int64_t i = 0; i < cnt; ++i) a[i] += p[i];
      } else {
        for (int64_t i = 0; i < cnt; ++i) acc[(size_t)i] += part[(size_t)i];
      }
    }
    for (int r = 0; r < world; ++r) {
      Rank& R = *g->ranks[(size_t)r];
      MCK(cudaSetDevice(R.dev));
      MCK(cudaMemcpyAsync(ptrs[(size_t)r], acc.data(), (size_t)cnt * elem, cudaMemcpyHostToDevice, R.stream));
      MCK(cudaStreamSynchronize(R.stream));
    }
  };
  std::vector<void*> ptrs((size_t)world);
  int64_t cnt = 0;
  fglt_error e{};
  for (int r = 0; r < world; ++r) {
    Rank& R = *g->ranks[(size_t)r];
    uint32_t* c3 = nullptr;
    stage_check(fglt_stage_triangles(R.ctx, b[(size_t)r][(size_t)r], b[(size_t)r][(size_t)r + 1],
                                     &c3, &cnt, &e), e, &(*outs)[(size_t)r]);
    ptrs[(size_t)r] = c3;
  }
  if (cnt && world > 1) host_sum(ptrs, cnt, 4);
  for (int r = 0; r < world; ++r) {
    Rank& R = *g->ranks[(size_t)r];
    uint64_t* c3v = nullptr;
    stage_check(fglt_stage_local_part(R.ctx, r, world, 0, &c3v, &cnt, &e), e,
                &(*outs)[(size_t)r]);
    ptrs[(size_t)r] = c3v;
  }
  if (cnt && world > 1) host_sum(ptrs, cnt, 8);
  for (int r = 0; r < world; ++r) {
    Rank& R = *g->ranks[(size_t)r];
    stage_check(fglt_stage_local_part(R.ctx, r, world, 1, nullptr, nullptr, &e), e,
                &(*outs)[(size_t)r]);
    uint64_t* vec = nullptr;
    stage_check(fglt_stage_roots(R.ctx, b[(size_t)r][(size_t)r], b[(size_t)r][(size_t)r + 1], &vec,
                                 &cnt, &e), e, &(*outs)[(size_t)r]);
    ptrs[(size_t)r] = vec;
  }
  if (cnt && world > 1) host_sum(ptrs, cnt, 8);
  for (int r = 0; r < world; ++r) rank_epilogue(g, r, j, &(*outs)[(size_t)r]);
}

}  // namespace

extern "C" int fglt_transform_multi(const int32_t* row_ptr, const int32_t* col_idx, int64_t n,
                                    int64_t nnz, uint32_t dict_mask, int lenient,
                                    const int* devices, int num_devices, uint32_t flags,
                                    uint64_t* raw_out, uint64_t* net_out, fglt_stats* stats,
                                    fglt_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (!devices || num_devices < 1) {
    put(err, FGLT_E_PARSE, "empty device list");
    return FGLT_E_PARSE;
  }
  if (dict_mask >> 16) {
    put(err, FGLT_E_PARSE, "graphlet id outside 0..15 in dictionary mask");
    return FGLT_E_PARSE;
  }
  if (n < 0 || nnz < 0 || n >= ((int64_t)1 << 31) || nnz >= ((int64_t)1 << 31) || nnz % 2) {
    put(err, FGLT_E_STRUCTURAL, "graph outside the int32 symmetric CSR limits");
    return FGLT_E_STRUCTURAL;
  }
  const int avail = fglt_device_count();
  for (int i = 0; i < num_devices; ++i)
    if (devices[i] < 0 || devices[i] >= avail) {
      put(err, FGLT_E_NO_DEVICE, "device " + std::to_string(devices[i]) + " not available (" +
                                     std::to_string(avail) + " devices); there is no CPU fallback");
      return FGLT_E_NO_DEVICE;
    }
  try {
    Group* g = group_for(devices, num_devices);
    std::lock_guard<std::mutex> lock(g->run);
    const int world = num_devices;
    Job j{row_ptr, col_idx, n, nnz, dict_mask | 3u, lenient, flags, raw_out, net_out, 0, {}};
    for (int i = 0; i < 16; ++i) j.k += (j.mask >> i) & 1u;
    for (int r = 0; r <= world; ++r) j.blocks.push_back(n * r / world);
    std::vector<Outcome> outs((size_t)world);
    std::vector<uint64_t> launches0((size_t)world);
    for (int r = 0; r < world; ++r)
      launches0[(size_t)r] = fglt_ctx_kernel_launches(g->ranks[(size_t)r]->ctx);
    if (g->emulated || world == 1) {
      try {
        run_emulated(g, j, &outs);
      } catch (const Fail& f) {
        bool any = false;
        for (auto& o : outs) any |= o.rc != 0;
        if (!any) {
          outs[0].rc = f.code;
          put(&outs[0].err, f.code, f.msg);
        }
      }
    } else {
      std::vector<std::thread> th;
      for (int r = 0; r < world; ++r) th.emplace_back(rank_nccl, g, r, &j, &outs[(size_t)r]);
      for (auto& t : th) t.join();
    }
    // the reference reports the first failure in (stage, vertex) order
    // (order_key 0: a failure outside the epilogue, e.g. CUDA, which wins)
    const Outcome* worst = nullptr;
    for (auto& o : outs)
      if (o.rc && (!worst || o.err.order_key < worst->err.order_key)) worst = &o;
    if (stats) {
      stats->device = devices[0];
      stats->threads_used = 1;  // host threads doing graphlet work: none (one driver thread per device)
      for (int r = 0; r < world; ++r)
        stats->kernel_launches +=
            fglt_ctx_kernel_launches(g->ranks[(size_t)r]->ctx) - launches0[(size_t)r];
    }
    if (worst) {
      if (err) *err = worst->err;
      return worst->rc;
    }
    return FGLT_OK;
  } catch (const Fail& f) {
    put(err, f.code, f.msg);
    return f.code;
  }
}
