// fglt_tables.h — the constant tables of the transform, defined ONCE and
// shared by the host API (graphlet_api.cpp) and the device pipeline
// (fglt.cu, fglt_roots.cuh):
//   * U16, the 16x16 unit upper-triangular net->raw coefficients (PAPER.md
//     Table 2; the reference's encoding proj/src/conversion.cpp:14-32), one
//     row packed 3 bits per column, usable as compile-time constants on host
//     and device;
//   * the reference's auxiliary steps in plan order with the graphlets that
//     need each (proj/src/dictionary.cpp:143-158) — the host's
//     resolve_dependencies and the device plan (make_plan) both read it.
#pragma once

#ifdef __CUDACC__
#define FGLT_HD __host__ __device__
#else
#define FGLT_HD
#endif

namespace fglt_tables {

FGLT_HD constexpr unsigned long long u16_row_packed(int r) {
  switch (r) {
    case 0: return 0x000000000001ull;
    case 1: return 0x000000000008ull;
    case 2: return 0x000000002040ull;
    case 3: return 0x000000001200ull;
    case 4: return 0x000000001000ull;
    case 5: return 0xca2050008000ull;
    case 6: return 0xd12440040000ull;
    case 7: return 0x650048200000ull;
    case 8: return 0x240201000000ull;
    case 9: return 0x610008000000ull;
    case 10: return 0xc90040000000ull;
    case 11: return 0x680200000000ull;
    case 12: return 0x649000000000ull;
    case 13: return 0x608000000000ull;
    case 14: return 0x640000000000ull;
    case 15: return 0x200000000000ull;
    default: return 0ull;
  }
}

// U16[r][c]: how many copies of net graphlet c contain raw graphlet r's orbit
FGLT_HD constexpr unsigned u16_coef(int r, int c) {
  return (unsigned)((u16_row_packed(r) >> (3 * c)) & 7ull);
}

constexpr unsigned id_bit(int id) { return 1u << id; }

// The reference's auxiliary steps, in plan order, with the dictionary ids
// that require each ("degrees" always runs).
struct AuxStepNeed {
  const char* name;
  unsigned needed_by;  // bit k set: graphlet k needs this step
};
constexpr int kNumAuxSteps = 7;
constexpr AuxStepNeed kAuxSteps[kNumAuxSteps] = {
    {"degrees", 0xFFFFu},
    {"triangles", id_bit(4) | id_bit(5) | id_bit(6) | id_bit(9) | id_bit(10) | id_bit(11) | id_bit(13)},
    {"two-paths", id_bit(2) | id_bit(5) | id_bit(6)},
    {"three-paths", id_bit(5)},
    {"four-cycle rows", id_bit(12) | id_bit(14)},
    {"diamond rows", id_bit(13)},
    {"tetrahedra", id_bit(15)},
};

}  // namespace fglt_tables
