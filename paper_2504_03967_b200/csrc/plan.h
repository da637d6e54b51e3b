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

struct HostOp {
    int kind;       // OpKind
    int t, c;       // register bits (-1 unused)
    int tq, cq;     // physical qubits (for export / debugging)
    uint64_t cmask, qmask;
    double m[8];
};

struct HostStage {
    std::vector<int> reg_tile, lane_tile, warp_tile;  // tile-bit index per register / lane / warp bit
    std::vector<HostOp> ops;
    bool tphase = false;
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
    int64_t n_ops = 0, n_stages = 0;
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
