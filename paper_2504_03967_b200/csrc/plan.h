// plan.h — host-side gate-fusion / remap planner (pure C++, no CUDA).
//
// Replaces the reference's per-gate dispatch (statevec.py:200-212 loop at
// :207-208) and per-gate LOCAL/EXCHANGE tagging (partition.py:100-109) with a
// program of fused passes: each pass streams the (shard of the) state once
// through the SMs in 2^k-amplitude tiles and applies every gate it holds in
// registers, with SMEM transposes between register stages.
#pragma once
#include <stdint.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/qgear_b200.h"
#include "desc.h"

namespace qg {

enum GateKindId { K_H = 0, K_RX = 1, K_RY = 2, K_RZ = 3, K_CX = 4, K_CR1 = 5, K_MEASURE = 6 };

struct Gate {
    int kind;
    int c, t;    // logical qubits (c = -1 for 1q kinds)
    double p;
    int64_t idx = -1;  // position in the circuit body (qg_plan_rebind)
};

// one register stage of a pass as scheduled (kept for qg_plan_rebind)
struct StageSched {
    std::vector<int> regs;   // physical register qubits demanded (<= rb)
    std::vector<Gate> gates; // executed in this order (physical qubits)
};

// a fused-kernel configuration: RB register bits, WB warp bits, k = RB + 5 + WB
struct KernelCfg {
    int id;
    int rb, wb;
    int k() const { return rb + kLaneBits + wb; }
};

// register-level op in slot coordinates (desc.h OpCode), planner output
enum AbsKind { A_RD = 0, A_CD = 1, A_PH = 2, A_CXM = 3, A_PH2 = 4, A_XF = 5, A_TPH = 6 };

struct HostOp {
    int kind;       // AbsKind
    int t, c;       // slot bits (-1 unused); A_XF: t = flip vector
    int form;       // A_RD / A_CD: 0 V = W = e_t; 1 V = e_t, W = e_t + e_c; 2 V = e_t + e_c, W = e_t
    int tq, cq;     // physical qubits (export / debugging)
    uint64_t cmask, qmask;  // thread predicate (all bits 1) / thread-phase select bit
    double m[8];    // A_RD: m00 m01 m10 m11; A_CD: 2x2 complex; A_PH2: e; A_TPH: v0, v1
    std::vector<std::pair<uint64_t, std::pair<double, double>>> ph;  // A_PH: (predicate, e) factors
    std::vector<std::pair<uint64_t, uint32_t>> xf;                    // A_XF: (predicate, flip vector) list
};

struct HostStage {
    std::vector<int> reg_tile, lane_tile, warp_tile;  // tile-bit index per register / lane / warp bit
    std::vector<HostOp> ops;       // kernel order (slot coordinates), excluding thread phases
    std::vector<HostOp> tph;       // thread-phase entries
    std::vector<uint32_t> out_vec; // per slot bit j: logical register-bit vector L^-1 e_j
};

struct HostPass {
    bool fused = true;
    KernelCfg cfg{};
    std::vector<int> tile_q;          // sorted physical positions, size k
    std::vector<HostStage> stages;
    HostStage io;
    bool load_direct = true, store_direct = true;
    GateOp gop{};                     // unfused single gate
    int n_gates = 0;                  // circuit gates covered by this pass
    int n_cxm = 0;                    // materialised register CX ops
    std::vector<StageSched> sched;    // the schedule this pass was emitted from
    Gate gate{};                      // unfused: the gate
    double gph_re = 1.0, gph_im = 0.0; // global phase factored out of this pass's diagonal ops
    bool scaled_rot = false;          // RD coefficients in the scaled form (Emitter::rotation)
    double rscale = 1.0;              // complex64: product of the scaled rotations' factors (applied
                                      // once, as an unconditional thread-phase entry at the pass end)
};

struct PlanStats {
    int64_t n_ops = 0, n_stages = 0, n_cxm = 0;
};

}  // namespace qg

namespace qg {
struct JitState;
}

struct qg_plan {
    int n = 0, n_local = 0, g = 0, dtype = 0;
    int64_t n_body = 0;
    qg::KernelCfg cfg{};
    std::vector<std::vector<qg::HostPass>> segs;
    std::vector<qg_remap> remaps;
    std::vector<int> final_phys;  // logical qubit -> physical position at the end
    qg::PlanStats stats;
    double gphase_re = 1.0, gphase_im = 0.0;  // global phase applied in the last fused pass
    std::vector<qg::Gate> body;       // validated circuit body (logical qubits), for rebind
    // device descriptors, built once at plan time (index = running fused-pass id)
    std::vector<qg::PassDesc<float>> d32;
    std::vector<qg::PassDesc<double>> d64;
    std::vector<std::vector<int64_t>> desc_index;  // [seg][pass] -> index into d32/d64 (-1 unfused)
    // circuit-specialised kernels of the d32 passes (jit.h), compiled asynchronously
    std::shared_ptr<qg::JitState> jit;
    int jit_threads = 0;
    int jit_mode = 0;  // qg_plan_opts.jit
    bool jit_blocking = true;  // false: tiered (interpreter until a pass's kernel is ready)
};

namespace qg {
// returns QG_OK or an error code; message in `err`
int build_plan(const int32_t* gate_type, const double* gate_param, int64_t n_gates, int n_qubits,
               const qg_plan_opts& opts, qg_plan& plan, std::string& err);
// new parameters for the same gate structure: re-emits every pass from its
// stored schedule (no rescheduling) and rebuilds the device descriptors
int rebind_plan(qg_plan& plan, const double* gate_param, int64_t n_gates, std::string& err);
}  // namespace qg
