// desc.h — device-side descriptors shared by the host planner (plan.cpp) and
// the fused-pass kernel (fused.cu).  A fused pass is passed BY VALUE as a
// __grid_constant__ kernel parameter (CUDA >= 12.1 allows 32 KiB of params),
// so every field below lives in the constant bank: warp-uniform, no global
// loads for the program.
#pragma once
#include <stdint.h>

namespace qg {

constexpr int kMaxStages = 8;    // register stages per pass (=> <= 7 SMEM transposes + io)
constexpr int kMaxOps = 128;     // register-level ops per pass
constexpr int kMaxMats = 128;    // coefficient sets per pass
constexpr int kLaneBits = 5;     // 32 lanes
constexpr int kMaxRegBits = 5;   // <= 32 amplitudes per thread
constexpr int kMaxWarpBits = 4;  // <= 16 warps per CTA
constexpr int kMaxTile = 16;     // tile qubits

// Register-level op kinds.  t/c are REGISTER bit indices inside the thread's
// 2^RB amplitudes; cmask is a set of GLOBAL index bits (lane/warp/tile-outside/
// rank bits) that must all be 1 for the op to act (thread-level control).
enum OpKind : uint8_t {
    OP_DENSE = 0,   // 2x2 complex on reg bit t                         m[0..7]
    OP_DIAG = 1,    // diag(d0, d1) on reg bit t                        m[0..3]
    OP_X = 2,       // swap the pairs of reg bit t                      —
    OP_CX = 3,      // swap pairs of reg bit t where reg bit c = 1      —
    OP_CPHASE = 4,  // amplitudes with reg bits t and c set *= e        m[0..1]
    OP_TPHASE = 5,  // thread phase: ph *= (gidx & qmask) ? v1 : v0    m[0..3]
};

struct OpDesc {
    uint8_t kind, t, c, pad;
    uint32_t mat;
    uint64_t cmask;
    uint64_t qmask;
};

// One register stage: the bijection (register bits, lane bits, warp bits) ->
// tile bits, expressed both as global qubit positions (for control/phase
// evaluation and global addresses) and as swizzled SMEM offsets (linear XOR
// swizzle, so the offset of a sum of bits is the XOR of their offsets).
struct StageDesc {
    uint16_t op_begin, op_end;
    uint8_t has_tphase, pad0;
    uint8_t reg_q[kMaxRegBits];
    uint8_t lane_q[kLaneBits];
    uint8_t warp_q[kMaxWarpBits];
    uint8_t pad1[2];
    uint16_t reg_s[kMaxRegBits];
    uint16_t lane_s[kLaneBits];
    uint16_t warp_s[kMaxWarpBits];
};

template <typename Real>
struct PassDesc {
    int32_t n_stages;      // compute stages (>= 1)
    int32_t k;             // tile qubits
    int32_t load_direct;   // 1: load with stage 0 mapping; 0: load with `io` then transpose
    int32_t store_direct;  // 1: store from the last stage; 0: transpose to `io` then store
    uint64_t n_tiles;      // 2^(n_local - k)
    uint8_t tile_q[kMaxTile];  // sorted physical positions of the tile bits
    // stg[0] = coalesced io mapping (lanes = tile bits 0..4); stg[1 + s] = compute stage s
    StageDesc stg[kMaxStages + 1];
    OpDesc ops[kMaxOps];
    Real mats[kMaxMats][8];
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
