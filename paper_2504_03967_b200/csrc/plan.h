// plan.h — host-side gate-fusion / remap planner (pure C++, no CUDA).
//
// Replaces the reference's per-gate dispatch (statevec.py:200-212 loop at
// :207-208) and per-gate LOCAL/EXCHANGE tagging (partition.py:100-109) with a
// program of fused passes: each pass streams the (shard of the) state once
// through the SMs in 2^k-amplitude tiles and applies every gate it holds in
// registers, with SMEM transposes between register stages.
#pragma once
#include <stdint.h>

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
};

// a fused-kernel configuration: RB register bits, WB warp bits, k = RB + 5 + WB
struct KernelCfg {
    int id;
    int rb, wb;
    int k() const { return rb + kLaneBits + wb; }
};

// abstract register-level op (planner output before round packing)
enum AbsKind { A_DENSE = 0, A_RDENSE = 1, A_DIAG = 2, A_X = 3, A_CX = 4, A_CP = 5, A_TPH = 6, A_CDIAG = 7 };

struct HostOp {
    int kind;       // AbsKind
    int t, c;       // register bits (-1 unused)
    int tq, cq;     // physical qubits (export / debugging)
    uint64_t cmask, qmask;
    double m[8];    // dense: 2x2 complex; rdense: m[0..3] real a00 a01 a10 a11;
                    // diag / tph: v0 = (m0,m1), v1 = (m2,m3); cp: (m0, m1)
};

struct HostRound {
    std::vector<HostOp> ops;  // in kernel slot-execution order
};

struct HostStage {
    std::vector<int> reg_tile, lane_tile, warp_tile;  // tile-bit index per register / lane / warp bit
    std::vector<HostOp> ops;       // program order (emitter output), excluding thread phases
    std::vector<HostOp> tph;       // thread-phase entries
    std::vector<HostRound> rounds; // packed
    std::vector<HostOp> deferred;  // register CX gates moved past the stage end (absorbed in out map)
    std::vector<uint32_t> out_vec; // per register bit: register-bit vector of its output tile index
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
};

struct PlanStats {
    int64_t n_ops = 0, n_stages = 0, n_rounds = 0;
};

}  // namespace qg

struct qg_plan {
    int n = 0, n_local = 0, g = 0, dtype = 0;
    int64_t n_body = 0;
    qg::KernelCfg cfg{};
    std::vector<std::vector<qg::HostPass>> segs;
    std::vector<qg_remap> remaps;
    std::vector<int> final_phys;  // logical qubit -> physical position at the end
    qg::PlanStats stats;
    // device descriptors, built once at plan time (index = running fused-pass id)
    std::vector<qg::PassDesc<float>> d32;
    std::vector<qg::PassDesc<double>> d64;
    std::vector<std::vector<int64_t>> desc_index;  // [seg][pass] -> index into d32/d64 (-1 unfused)
};

namespace qg {
// returns QG_OK or an error code; message in `err`
int build_plan(const int32_t* gate_type, const double* gate_param, int64_t n_gates, int n_qubits,
               const qg_plan_opts& opts, qg_plan& plan, std::string& err);
}  // namespace qg
