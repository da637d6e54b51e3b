// desc.h — device-side descriptors shared by the host planner (plan.cpp) and
// the fused-pass kernel (fused.cu).  A fused pass is passed BY VALUE as a
// __grid_constant__ kernel parameter (CUDA >= 12.1 allows 32 KiB of params),
// so every field below lives in the constant bank: warp-uniform, no global
// loads for the program.
//
// Program structure of one pass:
//   pass   = tile of k qubits (2^k amplitudes, one CTA at a time)
//   stage  = one register mapping (RB register bits, 5 lane bits, WB warp bits
//            -> tile bits); switching stage = one SMEM transpose
//   op     = one 32-bit word: body code (compile-time register bits baked in,
//            so the amplitude array is never indexed at run time), a thread
//            predicate index and a coefficient offset.  The kernel walks the
//            stage's op list and dispatches each word through one switch.
//
// Register layout inside a stage (what makes CX gates free): thread slot p
// holds the amplitude of logical register index i with
//        p = L i  xor  F
// L is a GF(2)-linear map shared by every thread (the register CX gates of the
// stage so far — the planner tracks it and never touches data for them), F a
// per-thread flip vector (X gates under a thread-level control: OC_XF).  The
// planner emits each op in slot coordinates; at the end of the stage the map
// (L, F) is folded into the transpose / store addresses (StageDesc.out_*).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define QG_HD __host__ __device__
#else
#define QG_HD
#endif

namespace qg {

constexpr int kMaxStages = 8;
constexpr int kMaxOps = 640;    // op words per pass
constexpr int kMaxTph = 128;    // thread-phase entries per pass
constexpr int kMaxPhe = 320;    // PH list entries per pass
constexpr int kMaxUph = 64;     // PH ops per pass with tile-uniform factors
constexpr int kMaxXfe = 256;    // XF list entries per pass
constexpr int kLaneBits = 5;
constexpr int kMaxRegBits = 6;
constexpr int kMaxWarpBits = 4;
constexpr int kMaxTile = 16;
template <typename Real>
struct CoefCap;
template <>
struct CoefCap<float> {
    static constexpr int value = 2560;  // coefficient reals per pass
};
template <>
struct CoefCap<double> {
    static constexpr int value = 1280;
};

// op word: bits 0-7 body code, 8-15 predicate index (0xff = none),
//          16-31 coefficient offset in reals / payload
//
// Pair ops act on slot pairs {p, p ^ V}; the member with parity(W & p) = 0 plays
// the logical |0> role (W . V = 1).  Standard ops have V = W = e_T; the W form
// (V = e_T, W = e_T + e_C) and the V form (V = e_T + e_C, W = e_T) cover the
// register qubits touched by an unexecuted register CX, so those need no moves.
// A thread whose flip vector F has parity(W & F) = 1 sees the roles swapped.
//
// Body codes are dense for the kernel's register width RB (one jump table):
//   fam 0 RD   + T            real 2x2, V = W = e_T          coef: m00 m01 m10 m11
//   fam 1 CD   + T            complex 2x2 (coef: 8 reals, row major)
//   fam 2 PH   + T            x e where parity(W & p) ^ f = 1, W = e_T; the phase is
//                             the product of a list of predicated entries (ph[]):
//                             word bits 8-14 = entry count, 15 = tile-uniform slot,
//                             16-31 = first entry;
//                             entry 0 is unconditional (its cmask is ignored)
//   fam 3 RDW, 4 RDV  + pair index (T, C)   the W / V forms of RD
//   fam 5 PHW  + tri index (T > C)   PH with W = e_T + e_C
//   fam 6 PH2  + tri index (T > C)   x e on logical |11> of slot bits (T, C); coef: e
//   OC_XF      (= oc_xf(RB)) a list of X gates under thread-level controls: for each
//              entry (xfe[]: control bit position | v << 8) F ^= v where that bit of
//              the thread's global index is 1; word bits 8-15 = entry count, 16-31 =
//              first entry
//   fam 7 CXM  + pair index (T, C) (after OC_XF): move slot p -> p ^ (p_C) e_T
//              (materialises part of L), F_T ^= F_C
//   OC_END     (= oc_end(RB)) terminates a stage's op list
enum OpFam { F_RD = 0, F_CD, F_PH, F_RDW, F_RDV, F_PHW, F_PH2 };
constexpr uint32_t kNoPred = 0xff;

QG_HD constexpr int oc_base(int fam, int rb) {
    return fam <= F_PH ? fam * rb
                       : (fam <= F_RDV ? 3 * rb + (fam - F_RDW) * rb * (rb - 1)
                                       : 3 * rb + 2 * rb * (rb - 1) + (fam - F_PHW) * rb * (rb - 1) / 2);
}
QG_HD constexpr int oc_std(int fam, int rb, int t) { return oc_base(fam, rb) + t; }
// OC_XF and the CXM family follow, so every code is a jump-table index
QG_HD constexpr uint32_t oc_xf(int rb) { return (uint32_t)(3 * rb + 3 * rb * (rb - 1)); }
QG_HD constexpr uint32_t oc_cxm(int rb, int t, int c) {
    return oc_xf(rb) + 1 + (uint32_t)(t * (rb - 1) + (c < t ? c : c - 1));
}
// ends every stage's op list
QG_HD constexpr uint32_t oc_end(int rb) { return oc_xf(rb) + 1 + (uint32_t)(rb * (rb - 1)); }
QG_HD constexpr int oc_pair(int fam, int rb, int t, int c) {
    return oc_base(fam, rb) + t * (rb - 1) + (c < t ? c : c - 1);
}
QG_HD constexpr int oc_tri(int fam, int rb, int t, int c) { return oc_base(fam, rb) + t * (t - 1) / 2 + c; }

QG_HD constexpr uint32_t op_word(uint32_t code, uint32_t pred, uint32_t coef) {
    return code | (pred << 8) | (coef << 16);
}

template <typename Real>
struct Entry {
    uint64_t cmask;      // global index bits that must all be 1
    uint64_t qmask;      // thread phase: bit selecting v1 over v0
    Real v[4];           // v0 = (v[0], v[1]), v1 = (v[2], v[3])
};

// one factor of an OC_PH phase: e where bit `pos` of the thread's global index
// is 1 (every predicate on this path is a single control qubit).  Entry 0 of a
// word's list is its unconditional factor; when word bit 15 is set its pad is the
// word's tile-uniform slot: the product of the word's factors whose control is a tile-id or
// rank bit (the same for every thread of a tile) is computed once per tile by one
// thread (PassDesc::uph) and read from shared memory by the op.
template <typename Real>
struct PhEnt {
    uint32_t pos;
    uint32_t pad;
    Real e[2];
};

struct StageDesc {
    uint16_t op_begin, op_end;
    uint16_t tph_begin, tph_end;  // thread-phase entries (applied after the ops)
    uint8_t reg_q[kMaxRegBits];
    uint8_t lane_q[kLaneBits];
    uint8_t warp_q[kMaxWarpBits];
    uint8_t pad[2];
    uint32_t reg_s[kMaxRegBits];   // input mapping: SMEM byte offset of each register bit
    uint16_t lane_s[kLaneBits];
    uint16_t warp_s[kMaxWarpBits];
    // output mapping (transpose out / global store): for slot bit j the tile-index
    // vector of L^-1 e_j (the stage's register CX gates, GF(2)-linear), as SMEM
    // offsets and as global index masks
    uint32_t out_s[kMaxRegBits];   // (SMEM byte offsets)
    uint64_t out_g[kMaxRegBits];
};

template <typename Real>
struct PassDesc {
    int32_t n_stages;      // compute stages (>= 1)
    int32_t k;             // tile qubits
    int32_t load_direct;   // 1: load with stage 0 mapping; 0: load with stg[0] (io) then transpose
    int32_t store_direct;  // 1: store from the last stage; 0: transpose to io then store
    int32_t tile_lo32;     // 1: every tile qubit < 32 (32-bit in-tile addressing)
    int32_t n_uph;         // tile-uniform phase slots (uph)
    uint64_t n_tiles;      // 2^(n_local - k)
    uint8_t tile_q[kMaxTile];  // sorted physical positions of the tile bits
    uint8_t comp_q[48];        // local positions outside the tile, ascending (tile id bits)
    // stg[0] = coalesced io mapping (lanes = tile bits 0..4); stg[1 + s] = compute stage s
    StageDesc stg[kMaxStages + 1];
    uint32_t ops[kMaxOps + 1];  // + 1: the kernel prefetches one word past a stage's list
    Entry<Real> tph[kMaxTph];
    PhEnt<Real> ph[kMaxPhe];
    uint32_t xfe[kMaxXfe];      // OC_XF list entries: control bit position | flip vector << 8
    Real coef[CoefCap<Real>::value];
    uint32_t uph[kMaxUph];      // tile-uniform slot: first ph entry | count << 16 (last: the
                                // other fields keep their constant-bank offsets)
};

// single-gate (unfused) op on global index bits
struct GateOp {
    int32_t kind;   // 0 = 2x2 on local target t under cmask; 1 = scale all amps by v under cmask/qmask
    int32_t t;
    uint64_t cmask;
    uint64_t qmask;
    double m[8];
};

}  // namespace qg
