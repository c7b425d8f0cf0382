// gen_main.cpp — `fglt_gen`, a standalone executable over the workload
// generators of gen.cpp: writes BASELINE.json config k as a raw int32 CSR
// (<prefix>.rp.i32, n+1 entries; <prefix>.ci.i32, nnz entries) and prints
// {"workload", "n", "nnz"} as one JSON line. bench.py's reference arm uses it
// so the process that times the reference never loads this package's
// libraries (it reads the files with numpy). Same instances as
// paper_2007_11111_b200/graphs.py CONFIGS.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

extern "C" {
int64_t fglt_build_csr32(const int64_t* eu, const int64_t* ev, int64_t ne, int64_t n,
                         int32_t* rp_out, int32_t* ci_out, int64_t* self_loops,
                         int64_t* dup_merged);
int64_t fglt_gen_er(int64_t n, double p, uint64_t seed, int64_t* eu, int64_t* ev);
int64_t fglt_gen_rmat(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                      int64_t* eu, int64_t* ev);
int64_t fglt_gen_rgg(int64_t n, double avg_deg, uint64_t seed, int64_t* eu, int64_t* ev);
int64_t fglt_gen_sbm(int64_t blocks, int64_t bs, double p_in, double cross_factor, uint64_t seed,
                     int64_t* eu, int64_t* ev);
}

namespace {

template <class F>
void two_pass(F f, std::vector<int64_t>* u, std::vector<int64_t>* v) {
  const int64_t k = f(nullptr, nullptr);
  u->resize((size_t)k);
  v->resize((size_t)k);
  f(u->data(), v->data());
}

bool write_all(const std::string& path, const void* p, size_t bytes) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) return false;
  const bool ok = std::fwrite(p, 1, bytes, f) == bytes;
  return std::fclose(f) == 0 && ok;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: fglt_gen CONFIG(1-5) OUT_PREFIX\n");
    return 2;
  }
  const int cfg = std::atoi(argv[1]);
  const std::string out = argv[2];
  std::vector<int64_t> u, v;
  int64_t n = 0;
  const char* name = nullptr;
  switch (cfg) {
    case 1:
      name = "er(n=2000,p=0.004,seed=1)";
      n = 2000;
      two_pass([](int64_t* a, int64_t* b) { return fglt_gen_er(2000, 0.004, 1, a, b); }, &u, &v);
      break;
    case 2:
      name = "rgg(n=2000000,avg_deg=3,seed=2,relabelled)";
      n = 2000000;
      two_pass([](int64_t* a, int64_t* b) { return fglt_gen_rgg(2000000, 3.0, 2, a, b); }, &u, &v);
      break;
    case 3:
    case 4: {
      const int scale = cfg == 3 ? 20 : 23;
      name = cfg == 3 ? "rmat(scale=20,ef=16,a=.57,b=.19,c=.19,seed=1)"
                      : "rmat(scale=23,ef=16,a=.57,b=.19,c=.19,seed=1)";
      n = int64_t{1} << scale;
      two_pass([scale](int64_t* a, int64_t* b) {
        return fglt_gen_rmat(scale, 16, 0.57, 0.19, 0.19, 1, a, b);
      }, &u, &v);
      break;
    }
    case 5:
      name = "sbm(blocks=65536,bs=64,p_in=0.3,cross=3n,seed=5)";
      n = int64_t{65536} * 64;
      two_pass([](int64_t* a, int64_t* b) { return fglt_gen_sbm(65536, 64, 0.3, 3.0, 5, a, b); },
               &u, &v);
      break;
    default:
      std::fprintf(stderr, "unknown config %d\n", cfg);
      return 2;
  }
  std::vector<int32_t> rp((size_t)n + 1), ci(std::max<size_t>(2 * u.size(), 1));
  int64_t loops = 0, dups = 0;
  const int64_t nnz =
      fglt_build_csr32(u.data(), v.data(), (int64_t)u.size(), n, rp.data(), ci.data(), &loops, &dups);
  if (!write_all(out + ".rp.i32", rp.data(), rp.size() * 4) ||
      !write_all(out + ".ci.i32", ci.data(), (size_t)nnz * 4)) {
    std::fprintf(stderr, "cannot write %s.*\n", out.c_str());
    return 5;
  }
  std::printf("{\"workload\": \"%s\", \"n\": %lld, \"nnz\": %lld}\n", name, (long long)n,
              (long long)nnz);
  return 0;
}
