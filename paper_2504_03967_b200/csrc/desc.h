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
//   round  = a FIXED sequence of slots, each bound to compile-time register
//            bits, enabled by bit masks (so the kernel never dispatches on a
//            runtime register index — that would force register-array copies):
//              1. 1q dense slots   b = 0..RB-1  (complex 2x2, or real 2x2)
//              2. diag slots       b = 0..RB-1  (thread-dependent diag(d0, d1):
//                                                 product of predicated entries)
//              3. X slots          b = 0..RB-1  (swap if an odd number of entry
//                                                 predicates hold)
//              4. CX slots         (t, c) register pairs
//              5. CPHASE slots     {t, c} register pairs
//   thread phase = product of predicated scalar entries over thread-level
//            qubits, applied once per stage (commutes with every slot).
#pragma once
#include <stdint.h>

namespace qg {

constexpr int kMaxStages = 8;
constexpr int kMaxRounds = 128;
constexpr int kMaxCoef = 96;
constexpr int kMaxEnt = 400;
constexpr int kLaneBits = 5;
constexpr int kMaxRegBits = 5;
constexpr int kMaxWarpBits = 4;
constexpr int kMaxTile = 16;

struct RoundDesc {
    uint8_t dense;       // complex 2x2 on reg bit b       (coef: 8 reals)
    uint8_t rdense;      // real 2x2 on reg bit b          (coef: 4 reals)
    uint8_t cdiag;       // constant diag(d0, d1) on reg bit b (coef: 4 reals)
    uint8_t diag;        // predicated diag slot on reg bit b (dcnt[b] entries)
    uint8_t xs;          // X slot on reg bit b            (xcnt[b] entries): folded into the
                         // thread's register flip mask, no data movement
    uint32_t cx;         // bit 5*t + c: swap pairs of reg bit t where reg bit c = 1
    uint16_t cp;         // bit t*(t-1)/2 + c (t > c): amps with both bits *= coef
    uint8_t dhi;         // diag slots whose d0 == 1 for every entry (only the |1> half changes)
    uint8_t dcnt[kMaxRegBits];
    uint8_t xcnt[kMaxRegBits];
    uint16_t coef;       // first coef row: dense/rdense in bit order, cdiag in bit order, then cp
    uint16_t ent;        // first entry: diag entries (bit order), then X entries (bit order)
    uint16_t pad2;
};

template <typename Real>
struct Entry {
    uint64_t cmask;      // global index bits that must all be 1
    uint64_t qmask;      // thread phase: bit selecting v1 over v0
    Real v[4];           // v0 = (v[0], v[1]), v1 = (v[2], v[3])
};

struct StageDesc {
    uint16_t round_begin, round_end;
    uint16_t tph_begin, tph_end;  // thread-phase entries
    uint8_t reg_q[kMaxRegBits];
    uint8_t lane_q[kLaneBits];
    uint8_t warp_q[kMaxWarpBits];
    uint8_t pad[2];
    uint16_t reg_s[kMaxRegBits];   // input mapping: SMEM offset of each register bit
    uint16_t lane_s[kLaneBits];
    uint16_t warp_s[kMaxWarpBits];
    // output mapping (transpose out / global store): the register bits' tile-index
    // vectors after the stage's deferred register CX gates (a GF(2)-linear map),
    // as SMEM offsets and as global index masks
    uint16_t out_s[kMaxRegBits];
    uint64_t out_g[kMaxRegBits];
};

template <typename Real>
struct PassDesc {
    int32_t n_stages;      // compute stages (>= 1)
    int32_t k;             // tile qubits
    int32_t load_direct;   // 1: load with stage 0 mapping; 0: load with stg[0] (io) then transpose
    int32_t store_direct;  // 1: store from the last stage; 0: transpose to io then store
    uint64_t n_tiles;      // 2^(n_local - k)
    uint8_t tile_q[kMaxTile];  // sorted physical positions of the tile bits
    uint8_t comp_q[48];        // local positions outside the tile, ascending (tile id bits)
    // stg[0] = coalesced io mapping (lanes = tile bits 0..4); stg[1 + s] = compute stage s
    StageDesc stg[kMaxStages + 1];
    RoundDesc rounds[kMaxRounds];
    Real coef[kMaxCoef][8];
    Entry<Real> ent[kMaxEnt];
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
