// plan.cpp — gate-fusion + qubit-remap planner (host C++).
//
// Reference behaviour this replaces / must preserve:
//   statevec.py:187-197  trailing-MEASURE split, MeasureMidCircuitError
//   statevec.py:147-184  per-gate validation (IndexOutOfRange, SelfPair) and dispatch
//   statevec.py:97-110   half-angle 2x2 matrices (computed here in fp64, cast at the end
//                        like statevec.py:117)
//   partition.py:89-109  shard layout: top log2(P) qubits are global
//
// Algorithm:
//   1. gates are scheduled into passes; a pass owns a tile of k qubits (the 5
//      lowest always included for coalescing); within a pass, gates run in
//      register stages whose register qubits must hold every NON-DIAGONAL target;
//      diagonal gates and all controls may sit on any qubit (evaluated from
//      thread-level index bits).  Gates may be moved ahead of deferred gates they
//      commute with (on every shared qubit both act diagonally).
//   2. consecutive 1-qubit ops on one register qubit are multiplied into one 2x2
//      (fp64) before the cast.
//   3. with P ranks, a non-diagonal target on a global qubit triggers a qubit
//      remap (all-to-all) that swaps the needed global qubits with the top local
//      positions; the logical->physical map is tracked to the end.
#include "plan.h"

#include <algorithm>
#include <climits>
#include <cassert>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

namespace qg {

using cd = std::complex<double>;

struct M2 {
    cd a00{1, 0}, a01{0, 0}, a10{0, 0}, a11{1, 0};
};

static M2 mul(const M2& A, const M2& B) {  // A * B
    M2 r;
    r.a00 = A.a00 * B.a00 + A.a01 * B.a10;
    r.a01 = A.a00 * B.a01 + A.a01 * B.a11;
    r.a10 = A.a10 * B.a00 + A.a11 * B.a10;
    r.a11 = A.a10 * B.a01 + A.a11 * B.a11;
    return r;
}

// statevec.py:97-110 (fp64, half-angle)
static M2 gate_matrix(int kind, double p) {
    M2 m;
    if (kind == K_H) {
        const double r = 1.0 / std::sqrt(2.0);
        m.a00 = r; m.a01 = r; m.a10 = r; m.a11 = -r;
        return m;
    }
    const double h = p / 2.0, c = std::cos(h), s = std::sin(h);
    if (kind == K_RX) {
        m.a00 = c; m.a01 = cd(0, -s); m.a10 = cd(0, -s); m.a11 = c;
    } else if (kind == K_RY) {
        m.a00 = c; m.a01 = -s; m.a10 = s; m.a11 = c;
    } else {  // RZ = diag(e^{-i h}, e^{i h})
        m.a00 = cd(std::cos(-h), std::sin(-h)); m.a01 = 0; m.a10 = 0; m.a11 = cd(std::cos(h), std::sin(h));
    }
    return m;
}

static cd expi(double lam) { return cd(std::cos(lam), std::sin(lam)); }  // np.exp(1j*lam)

static void put(double* d, const M2& m) {
    d[0] = m.a00.real(); d[1] = m.a00.imag(); d[2] = m.a01.real(); d[3] = m.a01.imag();
    d[4] = m.a10.real(); d[5] = m.a10.imag(); d[6] = m.a11.real(); d[7] = m.a11.imag();
}

static bool is_diag(const Gate& g) { return g.kind == K_RZ || g.kind == K_CR1; }

// ------------------------------------------------------------------ validation
static int validate(const int32_t* gt, const double* gp, int64_t n_gates, int n, std::vector<Gate>& body,
                    std::string& err) {
    // trailing MEASURE block (statevec.py:187-197)
    int64_t first_measure = n_gates;
    for (int64_t i = 0; i < n_gates; ++i) {
        const int k = gt[3 * i];
        if (k < 0 || k > K_MEASURE) {
            err = "gate " + std::to_string(i) + ": kind id " + std::to_string(k) + " out of range";
            return QG_E_CORRUPT_TENSOR;
        }
        if (k == K_MEASURE && first_measure == n_gates) first_measure = i;
    }
    for (int64_t i = first_measure; i < n_gates; ++i)
        if (gt[3 * i] != K_MEASURE) {
            err = "MEASURE records must form a trailing block";
            return QG_E_MEASURE_MID_CIRCUIT;
        }
    body.clear();
    body.reserve(first_measure);
    for (int64_t i = 0; i < first_measure; ++i) {
        const int k = gt[3 * i], c = gt[3 * i + 1], t = gt[3 * i + 2];
        const double p = gp[i];
        if (k == K_CX || k == K_CR1) {  // _check_pair statevec.py:155-160
            for (int q : {c, t})
                if (q < 0 || q >= n) {
                    err = "gate " + std::to_string(i) + ": qubit " + std::to_string(q) + " out of range for " +
                          std::to_string(n) + " qubits";
                    return QG_E_INDEX_OUT_OF_RANGE;
                }
            if (c == t) {
                err = "gate " + std::to_string(i) + ": control == target == " + std::to_string(c);
                return QG_E_SELF_PAIR;
            }
        } else if (t < 0 || t >= n) {  // statevec.py:149-150
            err = "gate " + std::to_string(i) + ": target " + std::to_string(t) + " out of range for " +
                  std::to_string(n) + " qubits";
            return QG_E_INDEX_OUT_OF_RANGE;
        }
        if ((k == K_RX || k == K_RY || k == K_RZ || k == K_CR1) && !std::isfinite(p)) {
            err = "gate " + std::to_string(i) + ": non-finite parameter";
            return QG_E_NONFINITE_PARAM;
        }
        body.push_back(Gate{k, (k == K_CX || k == K_CR1) ? c : -1, t, p, i});
    }
    return QG_OK;
}

// ------------------------------------------------------------------ kernel configs
// must match launch_fused in fused.cu
// auto choice = first entry with >= 8 qubits outside the tile; kernel_cfg (1 + id)
// forces one (tuning)
// (ids must match launch_fused in fused.cu; array index = id)
static const KernelCfg kCfgC64[] = {{0, 4, 4}, {1, 4, 3}, {2, 4, 2}, {3, 3, 0}, {4, 5, 3}, {5, 5, 4}, {6, 5, 2},
                                    {7, 6, 3}, {8, 6, 2}};
static const KernelCfg kCfgC128[] = {{0, 4, 3}, {1, 3, 2}, {2, 3, 0}, {3, 5, 3}};
// auto preference order (ids)
static const int kAutoC64[] = {4, 1, 2, 3};
static const int kAutoC128[] = {3, 0, 1, 2};

static bool pick_cfg(int dtype, int n_local, int force_k, int force_cfg, KernelCfg& out) {
    const KernelCfg* cfgs = dtype == QG_DTYPE_C64 ? kCfgC64 : kCfgC128;
    const int n_all = dtype == QG_DTYPE_C64 ? 9 : 4;
    const int* order = dtype == QG_DTYPE_C64 ? kAutoC64 : kAutoC128;
    const int nc = 4;  // auto candidates per dtype
    if (force_cfg > 0) {
        if (force_cfg > n_all || cfgs[force_cfg - 1].k() > n_local) return false;
        out = cfgs[force_cfg - 1];
        return true;
    }
    if (force_k > 0) {
        for (int i = 0; i < nc; ++i)
            if (cfgs[order[i]].k() == force_k && force_k <= n_local) { out = cfgs[order[i]]; return true; }
        return false;
    }
    // small states (measured on B200 with tools/probe_cfg.py, random CX-block circuits):
    // mid-size tiles beat the >= 256-tile rule below (c64 16-19 q: k = 11, 0.76 vs
    // 1.19 ms at 16 q; c128 16-17 q: k = 10, 0.85 vs 1.26 ms; c128 20 q: k = 13, 1.95 vs 2.13 ms)
    // (picked by tile size, so reordering the tables cannot change the choice)
    auto by_k = [&](int k) {
        for (int i = 0; i < nc; ++i)
            if (cfgs[order[i]].k() == k) { out = cfgs[order[i]]; return true; }
        return false;
    };
    if (dtype == QG_DTYPE_C64 && n_local >= 16 && n_local <= 19 && by_k(11)) return true;
    if (dtype == QG_DTYPE_C128 && n_local >= 16 && n_local <= 17 && by_k(10)) return true;
    if (dtype == QG_DTYPE_C128 && n_local == 20 && by_k(13)) return true;
    for (int i = 0; i < nc; ++i)
        if (n_local - cfgs[order[i]].k() >= 8) { out = cfgs[order[i]]; return true; }
    for (int i = 0; i < nc; ++i)
        if (cfgs[order[i]].k() <= n_local) { out = cfgs[order[i]]; return true; }
    return false;
}

// ------------------------------------------------------------------ scheduling
// per-qubit blocking state left by deferred gates: 0 free, 1 only diagonal
// actions may pass, 2 nothing may pass.
struct Blocks {
    std::vector<uint8_t> s;
    explicit Blocks(int n) : s(n, 0) {}
    bool blocked(const Gate& g) const {
        switch (g.kind) {
            case K_CX: return s[g.c] == 2 || s[g.t] != 0;
            case K_CR1: return s[g.c] == 2 || s[g.t] == 2;
            case K_RZ: return s[g.t] == 2;
            default: return s[g.t] != 0;
        }
    }
    void defer(const Gate& g) {
        auto z = [&](int q) { if (s[q] == 0) s[q] = 1; };
        switch (g.kind) {
            case K_CX: s[g.t] = 2; z(g.c); break;
            case K_CR1: z(g.c); z(g.t); break;
            case K_RZ: z(g.t); break;
            default: s[g.t] = 2;
        }
    }
};

// lanes pinned to the lowest tile bits in a coalesced (global load / store) mapping: 2 =
// every 32 B sector written / read whole by one warp access (QG_DEV_IOL: dev override;
// round 1 pinned all 5: 228 -> 202 transposes for the 32 q circuit, HBM time unchanged)
static const int kIoLanes = std::getenv("QG_DEV_IOL") ? std::atoi(std::getenv("QG_DEV_IOL")) : 2;

// per-amplitude instruction estimates; `in_reg` = register
// qubits of the stage being scanned (thread-level phases cost ~nothing per amp)
static double gate_cost(const Gate& g, const std::vector<char>& in_reg) {
    switch (g.kind) {
        case K_CX: return in_reg[g.c] ? 1.0 : 2.0;
        case K_CR1: {
            const int r = (in_reg[g.c] ? 1 : 0) + (in_reg[g.t] ? 1 : 0);
            return r == 2 ? 0.5 : (r == 1 ? 1.0 : 0.1);
        }
        case K_RZ: return in_reg[g.t] ? 2.0 : 0.1;
        case K_RX: return 9.0;
        default: return 5.0;  // H, RY: real 2x2
    }
}
constexpr double kStageCost = 6.0;

// Schedules one fused pass from `rem` (physical-qubit gates, valid order);
// leaves the unscheduled gates in `rem` (still a valid order).
static void schedule_pass(std::vector<Gate>& rem, int n, int n_local, int k, int rb, int c_low, int max_stages,
                          double max_cost, int max_gates, std::vector<int>& tile, std::vector<StageSched>& stages,
                          const std::vector<int>* fixed_tile = nullptr) {
    int n_taken = 0;
    std::vector<char> in_tile(n, 0);
    tile.clear();
    stages.clear();
    if (fixed_tile) {  // the tile is given (lookahead choice): stages pick registers inside it
        for (int q : *fixed_tile) { in_tile[q] = 1; tile.push_back(q); }
    } else {
        for (int q = 0; q < c_low && q < n_local; ++q) { in_tile[q] = 1; tile.push_back(q); }
    }
    double cost = 0;
    // one register stage: scan `rem` in order, execute what fits, defer the rest
    auto scan = [&](int s, bool restrict_low, StageSched& st, std::vector<Gate>& keep, double& scost) {
        Blocks B(n);
        std::vector<char> in_reg(n, 0);
        std::vector<int> tile_added;
        keep.clear();
        keep.reserve(rem.size());
        scost = s > 0 ? kStageCost : 0.0;
        bool stop = false;
        int n_x_blocked = 0;
        for (size_t i = 0; i < rem.size(); ++i) {
            const Gate& g = rem[i];
            if (stop) { keep.push_back(g); continue; }
            bool ok = false;
            if (!B.blocked(g)) {
                if (is_diag(g)) {
                    ok = true;
                } else {
                    const int t = g.t;
                    if (t < n_local) {
                        if (in_reg[t]) ok = true;
                        else if ((int)st.regs.size() < rb && (in_tile[t] || (int)tile.size() < k) &&
                                 !(restrict_low && t < kIoLanes)) {
                            in_reg[t] = 1;
                            st.regs.push_back(t);
                            if (!in_tile[t]) { in_tile[t] = 1; tile.push_back(t); tile_added.push_back(t); }
                            ok = true;
                        }
                    }
                }
            }
            if (ok && ((cost + scost + gate_cost(g, in_reg) > max_cost && !st.gates.empty()) ||
                       n_taken + (int)st.gates.size() >= max_gates)) {
                ok = false;
                stop = true;
            }
            if (ok) {
                st.gates.push_back(g);
                scost += gate_cost(g, in_reg);
            } else {
                if (!stop) {
                    const int before = B.s[g.t];
                    B.defer(g);
                    if (before != 2 && B.s[g.t] == 2 && ++n_x_blocked >= n) stop = true;
                }
                keep.push_back(g);
            }
        }
        if (st.gates.empty() && !fixed_tile) {  // undo tile growth of an empty stage
            for (int q : tile_added) { in_tile[q] = 0; tile.erase(std::find(tile.begin(), tile.end(), q)); }
        }
    };
    for (int s = 0; s < max_stages && !rem.empty(); ++s) {
        StageSched st;
        std::vector<Gate> keep;
        double scost = 0;
        // stage 0 keeps the pinned io-lane qubits out of registers so the tile
        // loads straight into the stage mapping; relax if that leaves it empty
        const bool restrict_low = s == 0 && c_low >= kLaneBits;
        scan(s, restrict_low, st, keep, scost);
        if (st.gates.empty() && restrict_low) {
            st = StageSched();
            scan(s, false, st, keep, scost);
        }
        if (st.gates.empty()) break;
        cost += scost;
        n_taken += (int)st.gates.size();
        rem.swap(keep);
        stages.push_back(std::move(st));
        if (cost >= max_cost || n_taken >= max_gates) break;
    }
    // fill the tile up to k qubits with the lowest unused local positions
    for (int q = 0; q < n_local && (int)tile.size() < k; ++q)
        if (!in_tile[q]) { in_tile[q] = 1; tile.push_back(q); }
    std::sort(tile.begin(), tile.end());
}

// Gates of `rem` (valid order) one pass over tile T could run, ignoring the register /
// stage / cost limits: a non-diagonal gate needs its target in T; blocked gates are
// deferred with the scheduler's rules (Blocks).  The tile search's objective.
static int tile_value(const std::vector<Gate>& rem, size_t window, const std::vector<char>& in_t, int n, int n_local) {
    Blocks B(n);
    int cnt = 0, n2 = 0;  // n2: qubits in state 2 (once all are, no later gate can run)
    const size_t m = std::min(window, rem.size());
    for (size_t i = 0; i < m && n2 < n; ++i) {
        const Gate& g = rem[i];
        if (!B.blocked(g) && (is_diag(g) || (g.t < n_local && in_t[g.t]))) {
            ++cnt;
            continue;
        }
        if (!is_diag(g) && B.s[g.t] != 2) ++n2;  // defer() sets a non-diagonal target to 2
        B.defer(g);
    }
    return cnt;
}

// Lookahead tile: start from the scheduler's first-come tile and swap free (non-low)
// tile qubits for other targets of the upcoming window while the number of runnable
// gates does not drop (deterministic pseudo-random local search).
static std::vector<int> search_tile(const std::vector<Gate>& rem, const std::vector<int>& start, int n, int n_local,
                                    int c_low, int iters, uint64_t seed) {
    static const size_t window = std::getenv("QG_DEV_TILE_WIN") ? (size_t)std::atoi(std::getenv("QG_DEV_TILE_WIN")) : 512;
    std::vector<char> in_t(n, 0);
    for (int q : start) in_t[q] = 1;
    std::vector<int> cand;  // non-diagonal targets in the window, outside the fixed low qubits
    {
        std::vector<char> seen(n, 0);
        for (size_t i = 0; i < std::min(window, rem.size()); ++i) {
            const Gate& g = rem[i];
            if (is_diag(g) || g.t >= n_local || g.t < c_low || seen[g.t]) continue;
            seen[g.t] = 1;
            cand.push_back(g.t);
        }
    }
    std::vector<int> freeq;
    for (int q : start)
        if (q >= c_low) freeq.push_back(q);
    if (freeq.empty() || cand.empty()) return start;
    int best = tile_value(rem, window, in_t, n, n_local);
    uint64_t x = seed * 0x9E3779B97F4A7C15ull + 1;
    auto rnd = [&](uint64_t m) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        return (size_t)(x % m);
    };
    for (int it = 0; it < iters; ++it) {
        const size_t ia = rnd(freeq.size());
        const int a = freeq[ia], b = cand[rnd(cand.size())];
        if (in_t[b]) continue;
        in_t[a] = 0;
        in_t[b] = 1;
        const int v = tile_value(rem, window, in_t, n, n_local);
        if (v >= best) {
            best = v;
            freeq[ia] = b;
        } else {
            in_t[b] = 0;
            in_t[a] = 1;
        }
    }
    std::vector<int> out;
    for (int q = 0; q < n; ++q)
        if (in_t[q]) out.push_back(q);
    return out;
}

// ------------------------------------------------------------------ mapping
static int swz(int dtype, int j) {  // linear XOR swizzle of a tile index (amplitude units)
    if (dtype == QG_DTYPE_C64) return j ^ (((j >> 4) ^ (j >> 8) ^ (j >> 12)) & 15);
    return j ^ (((j >> 3) ^ (j >> 6) ^ (j >> 9) ^ (j >> 12)) & 7);
}

// register/lane/warp tile bits of one stage
static void assign_mapping(int dtype, const KernelCfg& cfg, const std::vector<int>& reg_bits_needed, bool io_lanes,
                           HostStage& hs) {
    const int k = cfg.k();
    std::vector<char> used(k, 0);
    hs.reg_tile.clear(); hs.lane_tile.clear(); hs.warp_tile.clear();
    for (int b : reg_bits_needed) { hs.reg_tile.push_back(b); used[b] = 1; }
    if (io_lanes) {
        // coalesced: lanes 0..3 on tile bits 0..3 (every warp access is whole 128 B
        // lines of >= 256 B HBM runs), the fifth lane on the lowest free tile bit
        for (int l = 0; l < kIoLanes; ++l) { hs.lane_tile.push_back(l); used[l] = 1; }
        for (int b = kIoLanes; b < k && (int)hs.lane_tile.size() < kLaneBits; ++b)
            if (!used[b]) { hs.lane_tile.push_back(b); used[b] = 1; }
        for (int b = kLaneBits; b < k && (int)hs.reg_tile.size() < cfg.rb; ++b)
            if (!used[b]) { hs.reg_tile.push_back(b); used[b] = 1; }
    } else {
        // conflict-free lanes: the lanes of one SMEM wavefront must cover every
        // residue class of the swizzle (8B amps: 16-lane phases, 4 classes mod 4;
        // 16B amps: 8-lane phases, 3 classes mod 3), so the register fill (top bits
        // first) skips a bit whose class would be left without an unused member
        const int M = dtype == QG_DTYPE_C64 ? 4 : 3;
        auto spare = [&](int b) {
            int c = 0;
            for (int x = b % M; x < k; x += M) c += (!used[x] && x != b) ? 1 : 0;
            return c;
        };
        for (int b = k - 1; b >= 0 && (int)hs.reg_tile.size() < cfg.rb; --b)
            if (!used[b] && spare(b) >= 1) { hs.reg_tile.push_back(b); used[b] = 1; }
        for (int b = k - 1; b >= 0 && (int)hs.reg_tile.size() < cfg.rb; --b)
            if (!used[b]) { hs.reg_tile.push_back(b); used[b] = 1; }
        for (int r = 0; r < M; ++r)
            for (int b = 0; b < k; ++b)
                if (!used[b] && b % M == r) { hs.lane_tile.push_back(b); used[b] = 1; break; }
        for (int b = 0; b < k && (int)hs.lane_tile.size() < kLaneBits; ++b)
            if (!used[b]) { hs.lane_tile.push_back(b); used[b] = 1; }
    }
    for (int b = 0; b < k; ++b)
        if (!used[b]) { hs.warp_tile.push_back(b); used[b] = 1; }
}

// Re-choose the warp bits of a stage (ordered) keeping its register bits: the lanes and
// warps only decide which threads hold which thread-level tile bits, so ops, registers
// and results do not change.  Lanes keep the stage's constraint (io: tile bits
// 0..kIoLanes-1 pinned; otherwise conflict-free residue classes, as assign_mapping).
static bool set_warps(int dtype, int k, HostStage& h, const std::vector<int>& W, bool io) {
    std::vector<char> used(k, 0);
    for (int b : h.reg_tile) used[b] = 1;
    for (int b : W) {
        if (b < 0 || b >= k || used[b]) return false;
        used[b] = 1;
    }
    std::vector<int> lanes;
    if (io) {
        for (int l = 0; l < kIoLanes; ++l) {
            if (used[l]) return false;
            lanes.push_back(l);
            used[l] = 1;
        }
    } else {
        const int M = dtype == QG_DTYPE_C64 ? 4 : 3;
        for (int r = 0; r < M; ++r) {
            int pick = -1;
            for (int b = 0; b < k && pick < 0; ++b)
                if (!used[b] && b % M == r) pick = b;
            if (pick < 0) return false;
            lanes.push_back(pick);
            used[pick] = 1;
        }
    }
    for (int b = 0; b < k && (int)lanes.size() < kLaneBits; ++b)
        if (!used[b]) { lanes.push_back(b); used[b] = 1; }
    for (int b = 0; b < k; ++b)
        if (!used[b]) return false;
    h.lane_tile = lanes;
    h.warp_tile = W;
    return true;
}

// Sticky warp bits: consecutive mappings of a pass that place the same tile bits on the
// same warp-index bits hand data over inside each warp at the transpose (the kernels
// then synchronise the warp, or the warp pair when one warp bit changes, instead of
// the CTA; jit.cpp hand_sync).  The SMEM hand-overs of a tile form a cycle over the
// mappings (io load -> stage 0 -> ... -> last stage -> io store, the next tile's first
// transpose waiting on the previous tile's last reads), so the warp-bit sets are chosen
// by a DP around that cycle (cost 0 same set, 1 one bit differs, 4 otherwise), then
// ordered so that shared bits keep their warp index.
static void sticky_warps(int dtype, const KernelCfg& cfg, HostPass& hp, const std::vector<char>& io) {
    const int k = cfg.k(), S = (int)hp.stages.size(), WB = cfg.wb;
    if (WB <= 0 || S < 1) return;
    const bool use_io = !io[0] || !io[S - 1];
    std::vector<int> seq;  // node ids in hand-over order; S = the io mapping
    if (use_io) seq.push_back(S);
    for (int s = 0; s < S; ++s) seq.push_back(s);
    const int nn = (int)seq.size();
    if (nn < 2) return;
    auto bits_of = [&](uint32_t m) {
        std::vector<int> v;
        for (int b = 0; b < k; ++b)
            if (m >> b & 1u) v.push_back(b);
        return v;
    };
    std::vector<std::vector<uint32_t>> cand(nn);
    for (int i = 0; i < nn; ++i) {
        const int node = seq[i];
        for (uint32_t m = 0; m < (1u << k); ++m) {
            if (__builtin_popcount(m) != WB) continue;
            bool ok;
            if (node == S) {
                ok = (m & ((1u << kIoLanes) - 1)) == 0;
            } else {
                HostStage t = hp.stages[node];
                ok = set_warps(dtype, k, t, bits_of(m), io[node]);
            }
            if (ok) cand[i].push_back(m);
        }
        if (cand[i].empty()) return;  // keep assign_mapping's choice
    }
    auto cost = [](uint32_t a, uint32_t b) {
        const int d = __builtin_popcount(a ^ b) / 2;
        return d == 0 ? 0 : d == 1 ? 1 : 4;
    };
    int best = 1 << 30;
    std::vector<uint32_t> pick;
    for (uint32_t f : cand[0]) {
        std::vector<std::vector<int>> dp(nn), from(nn);
        dp[0].assign(cand[0].size(), 1 << 30);
        from[0].assign(cand[0].size(), -1);
        for (size_t j = 0; j < cand[0].size(); ++j)
            if (cand[0][j] == f) dp[0][j] = 0;
        for (int i = 1; i < nn; ++i) {
            dp[i].assign(cand[i].size(), 1 << 30);
            from[i].assign(cand[i].size(), -1);
            for (size_t j = 0; j < cand[i].size(); ++j)
                for (size_t p = 0; p < cand[i - 1].size(); ++p) {
                    if (dp[i - 1][p] >= (1 << 30)) continue;
                    const int c = dp[i - 1][p] + cost(cand[i - 1][p], cand[i][j]);
                    if (c < dp[i][j]) { dp[i][j] = c; from[i][j] = (int)p; }
                }
        }
        for (size_t j = 0; j < cand[nn - 1].size(); ++j) {
            if (dp[nn - 1][j] >= (1 << 30)) continue;
            const int c = dp[nn - 1][j] + cost(cand[nn - 1][j], f);
            if (c < best) {
                best = c;
                pick.assign(nn, 0);
                int jj = (int)j;
                for (int i = nn - 1; i >= 0; --i) {
                    pick[i] = cand[i][jj];
                    jj = from[i][jj];
                }
            }
        }
        if (best == 0) break;
    }
    if (pick.empty()) return;
    // order: shared bits keep the previous node's warp index, new bits fill the rest
    std::vector<int> prev;
    for (int i = 0; i < nn; ++i) {
        std::vector<int> W(WB, -1);
        std::vector<int> nb;
        for (int b : bits_of(pick[i])) {
            int at = -1;
            for (int j = 0; j < (int)prev.size(); ++j)
                if (prev[j] == b) at = j;
            if (at >= 0) W[at] = b; else nb.push_back(b);
        }
        for (int j = 0, t = 0; j < WB; ++j)
            if (W[j] < 0) W[j] = nb[t++];
        const int node = seq[i];
        if (node == S) {
            std::vector<char> used(k, 0);
            for (int b : W) used[b] = 1;
            std::vector<int> lanes, regs;
            for (int l = 0; l < kIoLanes; ++l) { lanes.push_back(l); used[l] = 1; }
            for (int b = kIoLanes; b < k && (int)lanes.size() < kLaneBits; ++b)
                if (!used[b]) { lanes.push_back(b); used[b] = 1; }
            for (int b = 0; b < k; ++b)
                if (!used[b]) regs.push_back(b);
            hp.io.lane_tile = lanes;
            hp.io.warp_tile = W;
            hp.io.reg_tile = regs;
        } else {
            HostStage& h = hp.stages[node];
            if (!set_warps(dtype, k, h, W, io[node])) return;  // (cannot happen: feasibility is order-free)
        }
        prev = W;
    }
}

// dev knob, off: measured on the 32 q circuit (profiles/r02i_sticky.jsonl) the sticky
// mappings move warp bits onto low tile bits, the load / store lanes then span 32 B sectors
// instead of 256 B runs, and the pass gets slower (22.8 vs 17.8 ms); with the scoped
// barriers the decoupled warps are slower still (27.2 ms)
// complex64 rotations in the scaled two-FMA form (Emitter::rotation; the kernels read the RD
// coefficients of complex64 passes in that form)
static constexpr bool kScaledRot = true;
static const bool kStickyWarps = std::getenv("QG_DEV_STICKY") ? std::atoi(std::getenv("QG_DEV_STICKY")) != 0 : false;

static bool disjoint_low5(const std::vector<int>& bits) {
    for (int b : bits) if (b < kIoLanes) return false;
    return true;
}

// ------------------------------------------------------------------ op emission
// Converts a stage's gates (program order, physical qubits) to slot-coordinate
// ops (desc.h).  Register CX gates are never executed: they update the stage's
// GF(2) map L (slot p holds logical register index i with p = L i ^ F) and the
// kernel folds L into the transpose / store addresses at the stage end.  An op
// on logical register bit b is emitted on slot bit T when L e_b = e_T and row b
// of L^-1 is e_T (diagonal ops only need the latter); otherwise L is first
// materialised by OC_CXM register moves (Gaussian elimination).
// Consecutive 1-qubit gates on one register qubit are multiplied in fp64 into
// at most [real 2x2][diag] factors (cheapest kernel ops: 2 + 1 FMA/amp) or one
// complex 2x2; diagonal factors are split into diag(1, e) and a global phase
// that the plan applies once (its last stage's thread-phase list).
static bool m_diag(const M2& m) { return m.a01 == cd(0) && m.a10 == cd(0); }
static bool m_real(const M2& m) {
    return m.a00.imag() == 0 && m.a01.imag() == 0 && m.a10.imag() == 0 && m.a11.imag() == 0;
}
static bool m_ident(const M2& m) { return m.a00 == cd(1) && m.a11 == cd(1) && m.a01 == cd(0) && m.a10 == cd(0); }

struct Emitter {
    HostStage& hs;
    const std::vector<int>& tile_q;
    const int rb;
    cd& gphase;
    std::vector<int> reg_of;  // physical qubit -> logical register bit or -1
    uint32_t row[kMaxRegBits];  // L as rows over logical bits
    std::vector<std::vector<M2>> pend;  // per logical bit: factors in application order
    // pending phases in SLOT coordinates, grouped by role vector W (one or two slot
    // bits): entries (predicate, e) applied as ONE OC_PH op.  Lazy register CX gates
    // move no data, so a queued phase survives them; a group is emitted only before
    // an op that does not commute with it (pair vector or flip vector v with
    // parity(W & v) = 1, or a CXM move) or at the stage end.
    std::vector<std::pair<uint32_t, std::vector<std::pair<uint64_t, cd>>>> sq;
    int n_cxm = 0;
    const bool scaled;   // complex64: rotations in the scaled two-FMA form (rotation())
    double rscale = 1.0; // product of their factors in this stage
    Emitter(HostStage& h, const std::vector<int>& tq, int n, int rb_, cd& gp, bool scaled_)
        : hs(h), tile_q(tq), rb(rb_), gphase(gp), reg_of(n, -1), pend(h.reg_tile.size()), scaled(scaled_) {
        for (size_t b = 0; b < hs.reg_tile.size(); ++b) reg_of[tile_q[hs.reg_tile[b]]] = (int)b;
        for (int r = 0; r < kMaxRegBits; ++r) row[r] = 1u << r;
    }
    int qphys(int b) const { return tile_q[hs.reg_tile[b]]; }
    // rows of L^-1
    void inverse(uint32_t* inv) const {
        uint32_t a[kMaxRegBits];
        for (int r = 0; r < rb; ++r) { a[r] = row[r]; inv[r] = 1u << r; }
        for (int j = 0; j < rb; ++j) {
            int p = j;
            while (!((a[p] >> j) & 1u)) ++p;
            std::swap(a[p], a[j]); std::swap(inv[p], inv[j]);
            for (int r = 0; r < rb; ++r)
                if (r != j && ((a[r] >> j) & 1u)) { a[r] ^= a[j]; inv[r] ^= inv[j]; }
        }
    }
    uint32_t col(int b) const {  // L e_b as a slot-bit vector
        uint32_t v = 0;
        for (int r = 0; r < rb; ++r) if ((row[r] >> b) & 1u) v |= 1u << r;
        return v;
    }
    // X gates under thread-level controls (F ^= v where pred) commute with every op
    // that does not read the F bits they flip: queue them and emit one OC_XF list op
    // before the first reader (or at the stage end) instead of one op each
    std::vector<std::pair<uint64_t, uint32_t>> xq;
    uint32_t xq_mask = 0;
    void flush_xf() {
        if (xq.empty()) return;
        for (const auto& x : xq) assert(x.first && !(x.first & (x.first - 1)));  // one control bit
        HostOp o{};
        o.kind = A_XF; o.t = (int)xq[0].second; o.c = -1; o.cmask = xq[0].first; o.tq = o.cq = -1;
        o.xf = xq;
        hs.ops.push_back(o);
        xq.clear();
        xq_mask = 0;
    }
    void push(int kind, int t, int c, uint64_t cmask = 0) {
        const uint32_t reads = (t >= 0 ? 1u << t : 0u) | (c >= 0 ? 1u << c : 0u);
        if (reads & xq_mask) flush_xf();
        HostOp o{};
        o.kind = kind; o.t = t; o.c = c; o.cmask = cmask;
        o.tq = (kind != A_XF && t >= 0) ? qphys(t) : -1;
        o.cq = c >= 0 ? qphys(c) : -1;
        hs.ops.push_back(o);
    }
    void materialise() {  // emit CXM row operations reducing L to the identity
        flush_phases(~0u);  // CXM moves data: queued phases go first
        for (int j = 0; j < rb; ++j) {
            if (!((row[j] >> j) & 1u)) {
                int i = j + 1;
                while (!((row[i] >> j) & 1u)) ++i;
                row[j] ^= row[i];
                push(A_CXM, j, i);
                ++n_cxm;
            }
            for (int i = 0; i < rb; ++i)
                if (i != j && ((row[i] >> j) & 1u)) {
                    row[i] ^= row[j];
                    push(A_CXM, i, j);
                    ++n_cxm;
                }
        }
    }
    static void inverse_of(const uint32_t* rows, int rb, uint32_t* inv) {
        uint32_t a[kMaxRegBits];
        for (int r = 0; r < rb; ++r) { a[r] = rows[r]; inv[r] = 1u << r; }
        for (int j = 0; j < rb; ++j) {
            int p = j;
            while (!((a[p] >> j) & 1u)) ++p;
            std::swap(a[p], a[j]); std::swap(inv[p], inv[j]);
            for (int r = 0; r < rb; ++r)
                if (r != j && ((a[r] >> j) & 1u)) { a[r] ^= a[j]; inv[r] ^= inv[j]; }
        }
    }
    // Fewest OC_CXM moves (<= 2, searched) that leave logical bit b in a form the
    // kernel has a body for (dense: V = W unit / W form / V form; phase: W with one
    // or two bits); applies them and returns true.  Full materialisation costs
    // rank(L - I) moves, usually 3.
    bool reduce_for(int b, bool dense) {
        auto form_ok = [&](const uint32_t* rows) {
            uint32_t inv[kMaxRegBits] = {};
            inverse_of(rows, rb, inv);
            const uint32_t w = inv[b];
            if (!dense) return unit(w) >= 0 || two(w);
            uint32_t v = 0;
            for (int r = 0; r < rb; ++r) if ((rows[r] >> b) & 1u) v |= 1u << r;
            return (unit(v) >= 0 && v == w) || (unit(v) >= 0 && two(w) && (w & v)) ||
                   (unit(w) >= 0 && two(v) && (w & v));
        };
        uint32_t r1[kMaxRegBits], r2[kMaxRegBits];
        int best[4] = {-1, -1, -1, -1};
        for (int t1 = 0; t1 < rb && best[0] < 0; ++t1)
            for (int c1 = 0; c1 < rb && best[0] < 0; ++c1) {
                if (t1 == c1) continue;
                std::memcpy(r1, row, sizeof(r1));
                r1[t1] ^= r1[c1];
                if (form_ok(r1)) { best[0] = t1; best[1] = c1; }
            }
        if (best[0] < 0)
            for (int t1 = 0; t1 < rb && best[0] < 0; ++t1)
                for (int c1 = 0; c1 < rb && best[0] < 0; ++c1) {
                    if (t1 == c1) continue;
                    std::memcpy(r1, row, sizeof(r1));
                    r1[t1] ^= r1[c1];
                    for (int t2 = 0; t2 < rb && best[0] < 0; ++t2)
                        for (int c2 = 0; c2 < rb && best[0] < 0; ++c2) {
                            if (t2 == c2) continue;
                            std::memcpy(r2, r1, sizeof(r2));
                            r2[t2] ^= r2[c2];
                            if (form_ok(r2)) { best[0] = t1; best[1] = c1; best[2] = t2; best[3] = c2; }
                        }
                }
        if (best[0] < 0) return false;
        flush_phases(~0u);  // CXM moves data: queued phases go first
        for (int k = 0; k < 4 && best[k] >= 0; k += 2) {
            row[best[k]] ^= row[best[k + 1]];
            push(A_CXM, best[k], best[k + 1]);
            ++n_cxm;
        }
        return true;
    }
    static int unit(uint32_t v) { return (v && !(v & (v - 1))) ? __builtin_ctz(v) : -1; }
    static bool two(uint32_t v) { return v && unit(v) < 0 && unit(v & (v - 1)) >= 0; }
    int slot_w(int b) {  // slot bit whose value is logical bit b (materialising if needed)
        uint32_t inv[kMaxRegBits] = {};
        inverse(inv);
        int t = unit(inv[b]);
        if (t < 0) { materialise(); t = b; }
        return t;
    }
    static bool odd(uint32_t x) { return __builtin_popcount(x) & 1; }
    // phase e on logical |1> of b (where the thread predicate cmask holds): queued
    // under its slot role vector W = row b of L^-1
    void emit_phase(int b, cd e, uint64_t cmask) {
        if (e == cd(1)) return;
        uint32_t inv[kMaxRegBits] = {};
        inverse(inv);
        uint32_t w = inv[b];
        if (unit(w) < 0 && !two(w)) {
            if (reduce_for(b, false)) { inverse(inv); w = inv[b]; }
            else { materialise(); w = 1u << b; }
        }
        for (auto& g : sq)
            if (g.first == w) { g.second.emplace_back(cmask, e); return; }
        sq.push_back({w, {{cmask, e}}});
    }
    void emit_group(const std::pair<uint32_t, std::vector<std::pair<uint64_t, cd>>>& g) {
        const uint32_t w = g.first;
        if (unit(w) >= 0) push(A_PH, unit(w), -1);
        else push(A_PH, 31 - __builtin_clz(w), __builtin_ctz(w));  // W form, T > C
        HostOp& o = hs.ops.back();
        cd e0(1, 0);  // the unconditional factors merged into entry 0
        for (const auto& x : g.second) if (!x.first) e0 *= x.second;
        o.ph.push_back({0, {e0.real(), e0.imag()}});
        for (const auto& x : g.second)
            if (x.first) o.ph.push_back({x.first, {x.second.real(), x.second.imag()}});
    }
    // emit the queued groups that do not commute with an op on slot vector v
    // (v = ~0: all of them), in queue order
    void flush_phases(uint32_t v) {
        std::vector<std::pair<uint32_t, std::vector<std::pair<uint64_t, cd>>>> keep;
        auto groups = std::move(sq);
        sq.clear();
        for (auto& g : groups) {
            if (v == ~0u || odd(g.first & v)) emit_group(g);
            else keep.push_back(std::move(g));
        }
        sq = std::move(keep);
    }
    void emit_diag(int b, const M2& m) {  // diag(d0, d1) = d0 * diag(1, d1 / d0)
        if (m.a00 != cd(1)) gphase *= m.a00;
        emit_phase(b, m.a11 / m.a00, 0);
    }
    // 2x2 on logical b: pairs along V = L e_b, roles by W = row b of L^-1; the kernel
    // has bodies for V = W = e_T, (V = e_T, W = e_T + e_C) and (V = e_T + e_C, W = e_T)
    // Real orthogonal 2x2 (H, RY and their products) as a rotation R(psi).  det -1:
    // M = Z R(psi), the Z is queued as a phase (usually merging with later phases on the
    // qubit); psi is folded into [-pi/2, pi/2] with R(psi + pi) = -R(psi) (sign -> global
    // phase).  complex64 (scaled): R(psi) = sigma * M with M = [[1, -t], [t, 1]], t = tan psi,
    // sigma = cos psi when |psi| <= pi/4 (form 0), else M = [[u, -1], [1, u]], u = cot psi,
    // sigma = sin psi (form 1): two FMAs per pair (x' = x - t y, y' = y + t x; x' = u x - y,
    // y' = x + u y); the factors sigma of a pass multiply into one real scale applied once at
    // its end (HostPass::rscale; they cannot be deferred further: each is in [1/sqrt2, 1]).
    // complex128: three in-place shears (Paeth: x += a y; y += b x; x += a y with
    // a = -tan(psi/2), b = sin psi), 3 FMAs per pair, no scale.
    bool rotation(const M2& m, double& a, double& bb, bool& refl, double& sigma) {
        const double m00 = m.a00.real(), m01 = m.a01.real(), m10 = m.a10.real(), m11 = m.a11.real();
        const double det = m00 * m11 - m01 * m10;
        refl = det < 0;
        // R = Z M when det = -1 (row 1 negated)
        const double r00 = m00, r01 = m01, r10 = refl ? -m10 : m10, r11 = refl ? -m11 : m11;
        double psi = std::atan2(r10, r00);
        const double c = std::cos(psi), s = std::sin(psi);
        const double e = std::fabs(c - r00) + std::fabs(s - r10) + std::fabs(-s - r01) + std::fabs(c - r11);
        if (e > 1e-12) return false;  // not orthogonal (never for products of H / RY)
        if (psi > M_PI / 2) { psi -= M_PI; gphase = -gphase; }
        else if (psi < -M_PI / 2) { psi += M_PI; gphase = -gphase; }
        sigma = 1.0;
        if (scaled) {
            const double cp = std::cos(psi), sp = std::sin(psi);
            if (std::fabs(sp) <= cp) { a = sp / cp; bb = 0.0; sigma = cp; }
            else { a = cp / sp; bb = 1.0; sigma = sp; }
            return true;
        }
        a = -std::tan(psi / 2);
        bb = std::sin(psi);
        return true;
    }
    void emit_dense(int b, const M2& m) {
        double ra = 0, rb_ = 0, sigma = 1.0;
        bool refl = false;
        const bool rot = m_real(m) && rotation(m, ra, rb_, refl, sigma);
        uint32_t inv[kMaxRegBits] = {};
        inverse(inv);
        uint32_t v = col(b), w = inv[b];
        const bool supported = (unit(v) >= 0 && v == w) || (rot && unit(v) >= 0 && two(w) && (w & v)) ||
                               (rot && unit(w) >= 0 && two(v) && (w & v));
        if (!supported && rot && reduce_for(b, true)) {
            inverse(inv);
            v = col(b);
            w = inv[b];
        }
        int t = -1, c = -1;
        if (unit(v) >= 0 && v == w) {
            t = unit(v);
        } else if (unit(v) >= 0 && two(w) && (w & v) && rot) {  // (no complex W/V bodies)
            t = unit(v); c = unit(w & ~v);
        } else if (unit(w) >= 0 && two(v) && (w & v) && rot) {
            t = unit(w); c = unit(v & ~w);
        } else {
            materialise();
            t = b; v = w = 1u << b;
        }
        flush_phases(v);  // phases acting on these pairs' members differently go first
        push(rot ? A_RD : A_CD, t, c);
        HostOp& o = hs.ops.back();
        o.form = c < 0 ? 0 : (v == (1u << t) ? 1 : 2);
        if (rot) {
            o.m[0] = ra;
            o.m[1] = rb_;
            rscale *= sigma;
            if (refl) emit_phase(b, cd(-1, 0), 0);  // Z after the rotation
        } else {
            put(o.m, m);
        }
    }
    void flush(int b) {
        std::vector<M2>& f = pend[b];
        if (f.empty()) return;
        auto cls = [](const M2& m) { return m_diag(m) ? 0 : (m_real(m) ? 1 : 2); };
        std::vector<M2> runs;  // runs of one class, merged (application order)
        for (const M2& m : f) {
            if (!runs.empty() && cls(runs.back()) == cls(m)) runs.back() = mul(m, runs.back());
            else runs.push_back(m);
        }
        f.clear();
        bool one = runs.size() > 2;
        for (const M2& m : runs) if (cls(m) == 2) one = true;
        if (one) {
            M2 u = runs[0];
            for (size_t i = 1; i < runs.size(); ++i) u = mul(runs[i], u);
            runs.assign(1, u);
        }
        for (const M2& m : runs) {
            if (m_ident(m)) continue;
            if (m_diag(m)) emit_diag(b, m);
            else emit_dense(b, m);
        }
    }
    void flush_nondiag(int b) {
        for (const M2& m : pend[b])
            if (!m_diag(m)) { flush(b); return; }
    }
    void tph(uint64_t cmask, uint64_t qmask, cd v0, cd v1) {
        HostOp o{};
        o.kind = A_TPH; o.t = o.c = o.tq = o.cq = -1;
        o.cmask = cmask; o.qmask = qmask;
        o.m[0] = v0.real(); o.m[1] = v0.imag(); o.m[2] = v1.real(); o.m[3] = v1.imag();
        hs.tph.push_back(o);
    }
    void gate(const Gate& g) {
        const int rt = reg_of[g.t];
        switch (g.kind) {
            case K_H: case K_RX: case K_RY:
                pend[rt].push_back(gate_matrix(g.kind, g.p));
                break;
            case K_RZ: {
                const M2 m = gate_matrix(K_RZ, g.p);
                if (rt >= 0) pend[rt].push_back(m);
                else tph(0, 1ull << g.t, m.a00, m.a11);
                break;
            }
            case K_CX: {
                flush(rt);
                const int rc = reg_of[g.c];
                if (rc >= 0) {
                    flush_nondiag(rc);
                    for (int r = 0; r < rb; ++r)  // L <- L * CX(c -> t)
                        if ((row[r] >> rt) & 1u) row[r] ^= 1u << rc;
                } else {
                    const uint32_t v = col(rt);  // slot vector now; stays valid past later lazy CX
                    flush_phases(v);
                    xq.emplace_back(1ull << g.c, v);
                    xq_mask |= v;
                }
                break;
            }
            case K_CR1: {
                const cd e = expi(g.p);
                const int rc = reg_of[g.c];
                if (rt >= 0 && rc >= 0) {
                    flush_nondiag(rt);
                    flush_nondiag(rc);
                    uint32_t inv[kMaxRegBits] = {};
                    inverse(inv);
                    if (unit(inv[rt]) < 0 || unit(inv[rc]) < 0) materialise();
                    const int a = slot_w(rt), b = slot_w(rc);  // both unit now
                    push(A_PH2, std::max(a, b), std::min(a, b));
                    hs.ops.back().m[0] = e.real(); hs.ops.back().m[1] = e.imag();
                } else if (rt >= 0 || rc >= 0) {
                    const int b = rt >= 0 ? rt : rc;
                    const int other = rt >= 0 ? g.c : g.t;
                    flush_nondiag(b);
                    emit_phase(b, e, 1ull << other);
                } else {
                    tph((1ull << g.t) | (1ull << g.c), 0, e, e);
                }
                break;
            }
            default: break;
        }
    }
    void finish() {
        for (size_t b = 0; b < pend.size(); ++b) flush((int)b);
        flush_phases(~0u);
        flush_xf();
        uint32_t inv[kMaxRegBits] = {};
        inverse(inv);
        hs.out_vec.assign(rb, 0);
        for (int j = 0; j < rb; ++j)  // column j of L^-1
            for (int b = 0; b < rb; ++b)
                if ((inv[b] >> j) & 1u) hs.out_vec[j] |= 1u << b;
    }
};

static HostPass make_fused_pass(int dtype, const KernelCfg& cfg, int n, const std::vector<int>& tile,
                                const std::vector<StageSched>& stages) {
    HostPass hp;
    hp.fused = true;
    hp.cfg = cfg;
    hp.tile_q = tile;
    std::vector<int> tbit(n, -1);
    for (size_t i = 0; i < tile.size(); ++i) tbit[tile[i]] = (int)i;
    const int S = (int)stages.size();
    hp.stages.resize(S);
    cd gphase(1, 0);
    hp.scaled_rot = kScaledRot && dtype == QG_DTYPE_C64;
    std::vector<char> io_s(S, 0);
    for (int s = 0; s < S; ++s) {
        std::vector<int> need;
        for (int q : stages[s].regs) need.push_back(tbit[q]);
        const bool compat = disjoint_low5(need);
        const bool io = compat && (s == 0 || s == S - 1);
        io_s[s] = io;
        assign_mapping(dtype, cfg, need, io, hp.stages[s]);
        Emitter em(hp.stages[s], hp.tile_q, n, cfg.rb, gphase, hp.scaled_rot);
        for (const Gate& g : stages[s].gates) em.gate(g);
        em.finish();
        hp.rscale *= em.rscale;
        hp.n_cxm += em.n_cxm;
        hp.n_gates += (int)stages[s].gates.size();
    }
    hp.gph_re = gphase.real();
    hp.gph_im = gphase.imag();
    auto is_io = [](const HostStage& h) {
        for (int l = 0; l < kIoLanes; ++l) if (h.lane_tile[l] != l) return false;
        return true;
    };
    hp.load_direct = is_io(hp.stages[0]);
    hp.store_direct = is_io(hp.stages[S - 1]);
    assign_mapping(dtype, cfg, {}, true, hp.io);
    if (kStickyWarps) sticky_warps(dtype, cfg, hp, io_s);
    hp.io.out_vec.assign(cfg.rb, 0);
    for (int b = 0; b < cfg.rb; ++b) hp.io.out_vec[b] = 1u << b;
    return hp;
}

static HostPass make_unfused_pass(const Gate& g, int n_local) {
    HostPass hp;
    hp.fused = false;
    hp.n_gates = 1;
    GateOp& o = hp.gop;
    std::memset(&o, 0, sizeof(o));
    auto local = [&](int q) { return q < n_local; };
    switch (g.kind) {
        case K_H: case K_RX: case K_RY: case K_RZ: {
            const M2 m = gate_matrix(g.kind, g.p);
            if (local(g.t)) { o.kind = 0; o.t = g.t; put(o.m, m); }
            else {  // RZ on a global qubit: per-rank scalar (H/RX/RY never reach here)
                o.kind = 1; o.qmask = 1ull << g.t;
                o.m[0] = m.a00.real(); o.m[1] = m.a00.imag(); o.m[2] = m.a11.real(); o.m[3] = m.a11.imag();
            }
            break;
        }
        case K_CX: {
            M2 x; x.a00 = 0; x.a01 = 1; x.a10 = 1; x.a11 = 0;
            o.kind = 0; o.t = g.t; o.cmask = 1ull << g.c; put(o.m, x);
            break;
        }
        case K_CR1: {
            const cd e = expi(g.p);
            if (local(g.t) || local(g.c)) {
                M2 d; d.a11 = e;
                o.kind = 0; o.t = local(g.t) ? g.t : g.c; o.cmask = 1ull << (local(g.t) ? g.c : g.t); put(o.m, d);
            } else {
                o.kind = 1; o.cmask = (1ull << g.c) | (1ull << g.t);
                o.m[0] = e.real(); o.m[1] = e.imag(); o.m[2] = e.real(); o.m[3] = e.imag();
            }
            break;
        }
    }
    return hp;
}

// ------------------------------------------------------------------ descriptors
static void fill_stage(int dtype, const HostPass& hp, const HostStage& h, StageDesc& d) {
    std::memset(&d, 0, sizeof(d));
    for (size_t b = 0; b < h.reg_tile.size(); ++b) {
        d.reg_q[b] = (uint8_t)hp.tile_q[h.reg_tile[b]];
        d.reg_s[b] = (uint32_t)swz(dtype, 1 << h.reg_tile[b]) * (dtype == QG_DTYPE_C64 ? 8u : 16u);
    }
    for (size_t b = 0; b < h.lane_tile.size(); ++b) {
        d.lane_q[b] = (uint8_t)hp.tile_q[h.lane_tile[b]];
        d.lane_s[b] = (uint16_t)swz(dtype, 1 << h.lane_tile[b]);
    }
    for (size_t b = 0; b < h.warp_tile.size(); ++b) {
        d.warp_q[b] = (uint8_t)hp.tile_q[h.warp_tile[b]];
        d.warp_s[b] = (uint16_t)swz(dtype, 1 << h.warp_tile[b]);
    }
    for (size_t b = 0; b < h.reg_tile.size(); ++b) {
        const uint32_t v = b < h.out_vec.size() ? h.out_vec[b] : (1u << b);
        int tidx = 0;
        uint64_t g = 0;
        for (size_t r = 0; r < h.reg_tile.size(); ++r)
            if (v & (1u << r)) {
                tidx |= 1 << h.reg_tile[r];
                g |= 1ull << hp.tile_q[h.reg_tile[r]];
            }
        d.out_s[b] = (uint32_t)swz(dtype, tidx) * (dtype == QG_DTYPE_C64 ? 8u : 16u);
        d.out_g[b] = g;
    }
}

template <typename Real>
static void put_entry(Entry<Real>& e, const HostOp& o) {
    e.cmask = o.cmask;
    e.qmask = o.qmask;
    for (int i = 0; i < 4; ++i) e.v[i] = (Real)o.m[i];
}

static int n_coef(const HostOp& o) {
    switch (o.kind) {
        case A_RD: return 2;
        case A_CD: return 8;
        case A_PH2: return 2;
        default: return 0;
    }
}

// resource needs of a pass (descriptor capacity is checked by the scheduler)
struct PassSize { int ops = 0, coef = 0, tph = 0, phe = 0, xfe = 0, uph = 0; };
static PassSize pass_size(const HostPass& hp) {
    PassSize z;
    for (const HostStage& h : hp.stages) {
        z.ops += (int)h.ops.size();
        z.tph += (int)h.tph.size();
        for (const HostOp& o : h.ops) {
            z.coef += n_coef(o);
            z.phe += (int)o.ph.size();
            z.xfe += (int)o.xf.size();
            if (o.kind == A_PH) {  // a tile-uniform slot when some control lies outside the tile
                bool uni = false;
                for (size_t i = 1; i < o.ph.size(); ++i)
                    uni |= std::find(hp.tile_q.begin(), hp.tile_q.end(), __builtin_ctzll(o.ph[i].first)) ==
                           hp.tile_q.end();
                z.uph += uni;
            }
        }
    }
    return z;
}

template <typename Real>
static bool fits_t(const HostPass& hp) {
    const PassSize z = pass_size(hp);
    // thread-phase slots kept free for the pass's rotation scale and the plan's global phase
    return z.ops + (int)hp.stages.size() <= kMaxOps && z.coef <= CoefCap<Real>::value && z.tph + 2 <= kMaxTph &&
           z.phe <= kMaxPhe && z.xfe <= kMaxXfe && z.uph <= kMaxUph;
}
static bool fits(int dtype, const HostPass& hp) {
    return dtype == QG_DTYPE_C64 ? fits_t<float>(hp) : fits_t<double>(hp);
}

static uint32_t op_code(const HostOp& o, int rb) {
    switch (o.kind) {
        case A_RD:
            return o.form == 0 ? oc_std(F_RD, rb, o.t) : oc_pair(o.form == 1 ? F_RDW : F_RDV, rb, o.t, o.c);
        case A_CD:
            return oc_std(F_CD, rb, o.t);  // complex ops only in the standard form
        case A_PH: return o.c < 0 ? oc_std(F_PH, rb, o.t) : oc_tri(F_PHW, rb, o.t, o.c);
        case A_PH2: return oc_tri(F_PH2, rb, o.t, o.c);
        case A_CXM: return oc_cxm(rb, o.t, o.c);
        default: return oc_xf(rb);
    }
}

template <typename Real>
static bool build_desc(const HostPass& hp, int n_local, PassDesc<Real>& d, std::string& err) {
    std::memset(&d, 0, sizeof(d));
    if (!fits_t<Real>(hp)) { err = "pass exceeds descriptor capacity"; return false; }
    const int dtype = sizeof(Real) == 4 ? QG_DTYPE_C64 : QG_DTYPE_C128;
    d.n_stages = (int)hp.stages.size();
    d.k = hp.cfg.k();
    d.load_direct = hp.load_direct;
    d.store_direct = hp.store_direct;
    d.n_tiles = 1ull << (n_local - d.k);
    for (int i = 0; i < d.k; ++i) d.tile_q[i] = (uint8_t)hp.tile_q[i];
    d.tile_lo32 = hp.tile_q.empty() || hp.tile_q.back() < 32 ? 1 : 0;  // tile_q is sorted
    {
        int nc0 = 0;
        for (int q = 0; q < n_local; ++q)
            if (std::find(hp.tile_q.begin(), hp.tile_q.end(), q) == hp.tile_q.end()) d.comp_q[nc0++] = (uint8_t)q;
    }
    fill_stage(dtype, hp, hp.io, d.stg[0]);
    int no = 0, nc = 0, nt = 0, nph = 0, nxf = 0;
    for (int s = 0; s < d.n_stages; ++s) {
        const HostStage& h = hp.stages[s];
        StageDesc& sd = d.stg[1 + s];
        fill_stage(dtype, hp, h, sd);
        sd.op_begin = (uint16_t)no;
        for (const HostOp& o : h.ops) {
            uint32_t w;
            if (o.kind == A_XF) {
                w = op_word(oc_xf(hp.cfg.rb), (uint32_t)o.xf.size(), (uint32_t)nxf);
                for (const auto& x : o.xf) d.xfe[nxf++] = (uint32_t)__builtin_ctzll(x.first) | (x.second << 8);
            } else if (o.kind == A_CXM) {
                w = op_word(oc_cxm(hp.cfg.rb, o.t, o.c), kNoPred, 0);
            } else if (o.kind == A_PH) {
                // entry 0, then the factors controlled by tile bits (per thread); the
                // factors controlled by tile-id / rank bits go to a tile-uniform slot
                // (word bits 8-14 = entry count, bit 15 = has a tile-uniform slot)
                std::vector<size_t> thr, uni;
                for (size_t i = 1; i < o.ph.size(); ++i) {
                    const int pos = __builtin_ctzll(o.ph[i].first);
                    (std::find(hp.tile_q.begin(), hp.tile_q.end(), pos) != hp.tile_q.end() ? thr : uni).push_back(i);
                }
                if (1 + thr.size() > 127) { err = "phase list too long"; return false; }
                w = op_word(op_code(o, hp.cfg.rb), (uint32_t)(1 + thr.size()) | (uni.empty() ? 0u : 0x80u),
                            (uint32_t)nph);
                auto put = [&](const std::pair<uint64_t, std::pair<double, double>>& x) {
                    d.ph[nph].pos = x.first ? (uint32_t)__builtin_ctzll(x.first) : 0u;
                    d.ph[nph].pad = 0;
                    d.ph[nph].e[0] = (Real)x.second.first;
                    d.ph[nph].e[1] = (Real)x.second.second;
                    ++nph;
                };
                const int e0 = nph;
                put(o.ph[0]);
                for (size_t i : thr) put(o.ph[i]);
                if (!uni.empty()) {
                    d.ph[e0].pad = (uint32_t)d.n_uph;
                    d.uph[d.n_uph++] = (uint32_t)nph | ((uint32_t)uni.size() << 16);
                    for (size_t i : uni) put(o.ph[i]);
                }
            } else {
                w = op_word(op_code(o, hp.cfg.rb), kNoPred, (uint32_t)nc);
                for (int i = 0; i < n_coef(o); ++i) d.coef[nc++] = (Real)o.m[i];
            }
            d.ops[no++] = w;
        }
        d.ops[no++] = op_word(oc_end(hp.cfg.rb), 0, 0);
        sd.op_end = (uint16_t)no;
        sd.tph_begin = (uint16_t)nt;
        for (const HostOp& o : h.tph) put_entry(d.tph[nt++], o);
        sd.tph_end = (uint16_t)nt;
    }
    return true;
}

// appends the plan's accumulated global phase to the last stage of a built descriptor
template <typename Real>
static void add_global_phase(PassDesc<Real>& d, cd g) {
    StageDesc& sd = d.stg[d.n_stages];
    Entry<Real>& e = d.tph[sd.tph_end];
    e.cmask = 0;
    e.qmask = 0;
    e.v[0] = e.v[2] = (Real)g.real();
    e.v[1] = e.v[3] = (Real)g.imag();
    sd.tph_end = (uint16_t)(sd.tph_end + 1);
}

// device descriptors of every pass, stats, and the plan's global phase
static int build_descriptors(qg_plan& plan, std::string& err) {
    cd gphase(1, 0);
    int64_t last_desc = -1;
    plan.d32.clear();
    plan.d64.clear();
    plan.desc_index.assign(plan.segs.size(), {});
    plan.stats = PlanStats{};
    for (size_t s = 0; s < plan.segs.size(); ++s) {
        for (const HostPass& hp : plan.segs[s]) {
            int64_t idx = -1;
            if (hp.fused) {
                gphase *= cd(hp.gph_re, hp.gph_im);
                if (plan.dtype == QG_DTYPE_C64) {
                    plan.d32.emplace_back();
                    if (!build_desc<float>(hp, plan.n_local, plan.d32.back(), err)) return QG_E_INVALID_ARG;
                    if (hp.rscale != 1.0) add_global_phase(plan.d32.back(), cd(hp.rscale, 0));
                    idx = (int64_t)plan.d32.size() - 1;
                } else {
                    plan.d64.emplace_back();
                    if (!build_desc<double>(hp, plan.n_local, plan.d64.back(), err)) return QG_E_INVALID_ARG;
                    idx = (int64_t)plan.d64.size() - 1;
                }
                last_desc = idx;
                plan.stats.n_stages += (int64_t)hp.stages.size();
                plan.stats.n_cxm += hp.n_cxm;
                for (const HostStage& h : hp.stages) plan.stats.n_ops += (int64_t)(h.ops.size() + h.tph.size());
            } else {
                plan.stats.n_ops += 1;
            }
            plan.desc_index[s].push_back(idx);
        }
    }
    if (last_desc >= 0 && gphase != cd(1, 0)) {
        if (plan.dtype == QG_DTYPE_C64) add_global_phase(plan.d32[last_desc], gphase);
        else add_global_phase(plan.d64[last_desc], gphase);
    }
    plan.gphase_re = gphase.real();
    plan.gphase_im = gphase.imag();
    return QG_OK;
}

int rebind_plan(qg_plan& plan, const double* gate_param, int64_t n_gates, std::string& err) {
    if (n_gates < plan.n_body || (plan.n_body > 0 && !gate_param)) {
        err = "rebind needs the parameters of all " + std::to_string(plan.n_body) + " body gates";
        return QG_E_INVALID_ARG;
    }
    for (int64_t i = 0; i < plan.n_body; ++i) {
        const int k = plan.body[i].kind;
        if ((k == K_RX || k == K_RY || k == K_RZ || k == K_CR1) && !std::isfinite(gate_param[i])) {
            err = "gate " + std::to_string(i) + ": non-finite parameter";
            return QG_E_NONFINITE_PARAM;
        }
    }
    for (int64_t i = 0; i < plan.n_body; ++i) plan.body[i].p = gate_param[i];
    for (auto& seg : plan.segs)
        for (HostPass& hp : seg) {
            if (hp.fused) {
                for (StageSched& st : hp.sched)
                    for (Gate& g : st.gates) g.p = gate_param[g.idx];
                HostPass fresh = make_fused_pass(plan.dtype, hp.cfg, plan.n, hp.tile_q, hp.sched);
                if (!fits(plan.dtype, fresh)) {
                    err = "rebound pass exceeds descriptor capacity (plan the circuit afresh)";
                    return QG_E_INVALID_ARG;
                }
                fresh.sched = std::move(hp.sched);
                hp = std::move(fresh);
            } else {
                Gate g = hp.gate;
                g.p = gate_param[g.idx];
                hp = make_unfused_pass(g, plan.n_local);
                hp.gate = g;
            }
        }
    return build_descriptors(plan, err);
}

// ------------------------------------------------------------------ driver
// lookahead tile search iterations per fused pass (0 = first-come tiles; QG_DEV_TILE_SEARCH)
static const int kTileSearch = std::getenv("QG_DEV_TILE_SEARCH") ? std::atoi(std::getenv("QG_DEV_TILE_SEARCH")) : 400;
// independent searches per pass (different seeds, evaluated on host threads; QG_DEV_TILE_K):
// 8 take the 32 q random circuit from 71 to 68 passes but not its time (1.232 -> 1.244 s: the
// fewer passes carry the same gates, and a pass's time now grows with its gates), so 1
static const int kTileStarts =
    std::getenv("QG_DEV_TILE_K") ? std::max(1, std::atoi(std::getenv("QG_DEV_TILE_K"))) : 1;
static int plan_threads() {
    static const int t = [] {
        const unsigned hw = std::thread::hardware_concurrency();
        return hw == 0 ? 1 : (int)std::min(hw, 8u);
    }();
    return t;
}

constexpr int kRemapMinPos = 10;  // 8 KiB runs (complex64) in a remap's strided blocks

int build_plan(const int32_t* gate_type, const double* gate_param, int64_t n_gates, int n_qubits,
               const qg_plan_opts& opts, qg_plan& plan, std::string& err) {
    if (n_qubits < 1 || n_qubits > 62) { err = "n_qubits must be in [1, 62]"; return QG_E_INVALID_ARG; }
    if (opts.dtype != QG_DTYPE_C64 && opts.dtype != QG_DTYPE_C128) { err = "bad dtype"; return QG_E_INVALID_ARG; }
    if (opts.log2_ranks < 0 || opts.log2_ranks > n_qubits || opts.log2_ranks > 8) {
        err = "workers must be a power of two <= 2^n_qubits (and <= 256)";
        return QG_E_BAD_WORKER_COUNT;
    }
    if (n_gates < 0 || (n_gates > 0 && (!gate_type || !gate_param))) { err = "bad gate arrays"; return QG_E_INVALID_ARG; }
    std::vector<Gate> body;
    int rc = validate(gate_type, gate_param, n_gates, n_qubits, body, err);
    if (rc != QG_OK) return rc;

    plan.n = n_qubits;
    plan.g = opts.log2_ranks;
    plan.n_local = n_qubits - opts.log2_ranks;
    plan.dtype = opts.dtype;
    plan.n_body = (int64_t)body.size();
    const int n = n_qubits, n_local = plan.n_local;

    KernelCfg cfg{};
    bool fused = opts.fuse != 0 && pick_cfg(opts.dtype, n_local, opts.tile_qubits, opts.kernel_cfg, cfg);
    if (opts.fuse != 0 && (opts.tile_qubits > 0 || opts.kernel_cfg > 0) && !fused) {
        err = "tile_qubits not available for this dtype / size";
        return QG_E_INVALID_ARG;
    }
    plan.cfg = cfg;
    const int max_stages = opts.max_stages > 0 ? std::min(opts.max_stages, kMaxStages) : kMaxStages;
    const double max_cost = opts.max_cost > 0 ? (double)opts.max_cost : 350.0;
    // small states live in L2: no coalescing constraint; large ones keep the lowest
    // c_low qubits in every tile, so each HBM access is a 2^c_low-amplitude run
    int c_low = n_local >= 20 ? kLaneBits : 0;
    if (const char* e = std::getenv("QG_DEV_CLOW")) c_low = std::atoi(e);  // dev probe only
    if (opts.low_qubits > 0 && n_local >= 20) c_low = std::min(std::max(opts.low_qubits, kLaneBits), cfg.k() - 1);

    std::vector<int> phys(n), inv(n);  // logical -> physical, physical -> logical
    for (int q = 0; q < n; ++q) phys[q] = inv[q] = q;

    std::vector<Gate> rem;  // physical-qubit gates still to run
    auto to_phys = [&](const std::vector<Gate>& logical) {
        std::vector<Gate> out(logical);
        for (Gate& g : out) { g.t = phys[g.t]; if (g.c >= 0) g.c = phys[g.c]; }
        return out;
    };
    std::vector<Gate> rem_logical = body;
    plan.segs.emplace_back();
    while (!rem_logical.empty()) {
        rem = to_phys(rem_logical);
        // passes of this segment
        while (!rem.empty()) {
            const size_t before = rem.size();
            if (fused) {
                std::vector<int> tile;
                std::vector<StageSched> stages;
                int max_gates = kMaxOps;  // shrunk below if the descriptor overflows
                HostPass hp;
                for (;;) {
                    std::vector<Gate> trial(rem);
                    schedule_pass(trial, n, n_local, cfg.k(), cfg.rb, c_low, max_stages, max_cost, max_gates,
                                  tile, stages);
                    if (stages.empty()) break;
                    if (kTileSearch > 0 && (int)tile.size() == cfg.k() && c_low > 0) {
                        // lookahead tile: keep it when its pass schedules more gates
                        static const uint64_t seed0 =
                            std::getenv("QG_DEV_TILE_SEED") ? std::strtoull(std::getenv("QG_DEV_TILE_SEED"), nullptr, 10) : 0;
                        // kTileStarts independent searches (seeds j), each scheduled; the pass
                        // keeps the one that schedules the most gates (ties: lowest j), so the
                        // plan does not depend on how many host threads evaluate them
                        struct Cand {
                            std::vector<Gate> trial;
                            std::vector<int> tile;
                            std::vector<StageSched> stages;
                            bool ok = false;
                        };
                        std::vector<Cand> cands(kTileStarts);
                        const uint64_t sbase = seed0 * 1000003 + plan.segs.back().size() + 7 * plan.segs.size();
                        auto eval = [&](int sj) {
                            const std::vector<int> t2 =
                                search_tile(rem, tile, n, n_local, c_low, kTileSearch, sbase + (uint64_t)sj * 7919);
                            if (t2 == tile) return;
                            Cand& c = cands[sj];
                            c.trial = rem;
                            schedule_pass(c.trial, n, n_local, cfg.k(), cfg.rb, c_low, max_stages, max_cost, max_gates,
                                          c.tile, c.stages, &t2);
                            c.ok = !c.stages.empty();
                        };
                        const int nth = std::min(kTileStarts, plan_threads());
                        std::vector<std::thread> th;
                        for (int w = 1; w < nth; ++w)
                            th.emplace_back([&, w] { for (int sj = w; sj < kTileStarts; sj += nth) eval(sj); });
                        for (int sj = 0; sj < kTileStarts; sj += nth) eval(sj);
                        for (auto& t : th) t.join();
                        for (Cand& c : cands)
                            if (c.ok && c.trial.size() < trial.size()) {
                                trial.swap(c.trial);
                                tile.swap(c.tile);
                                stages.swap(c.stages);
                            }
                    }
                    hp = make_fused_pass(opts.dtype, cfg, n, tile, stages);
                    if (fits(opts.dtype, hp) || max_gates <= 1) { rem.swap(trial); break; }
                    max_gates = std::max(1, hp.n_gates * 3 / 4);
                }
                if (stages.empty()) break;
                if (std::getenv("QG_DEV_PLAN_DUMP")) {  // dev probe: tile qubits per pass
                    std::fprintf(stderr, "tile");
                    for (int q : tile) std::fprintf(stderr, " %d", q);
                    std::fprintf(stderr, "\n");
                }
                hp.sched = stages;
                plan.segs.back().push_back(std::move(hp));
            } else {
                const Gate& g = rem.front();
                if (!is_diag(g) && g.t >= n_local) break;
                plan.segs.back().push_back(make_unfused_pass(g, n_local));
                plan.segs.back().back().gate = g;
                rem.erase(rem.begin());
            }
            if (rem.size() == before) break;
        }
        // back to logical for the remap decision
        rem_logical = rem;
        for (Gate& g : rem_logical) { g.t = inv[g.t]; if (g.c >= 0) g.c = inv[g.c]; }
        if (rem_logical.empty()) break;
        // qubit remap: bring in the global positions needed soonest (Belady order)
        std::vector<int> need;
        for (const Gate& g : rem_logical) {
            if (is_diag(g)) continue;
            const int p = phys[g.t];
            if (p >= n_local && std::find(need.begin(), need.end(), p) == need.end()) need.push_back(p);
            // at most min(g, n_local) qubits per remap: they swap with the top local positions
            if ((int)need.size() == std::min(plan.g, n_local)) break;
        }
        if (n_local == 0) {  // no local position to swap a global target into
            err = "workers = 2^n_qubits leaves no local qubit for a non-diagonal gate";
            return QG_E_BAD_WORKER_COUNT;
        }
        if (need.empty()) { err = "planner made no progress"; return QG_E_PROTOCOL; }
        qg_remap rm{};
        rm.s = (int)need.size();
        // Belady eviction: the s local qubits whose next use as a non-diagonal target
        // is furthest away (never used again first) go global; ties prefer higher
        // positions (longer contiguous runs in the exchange's strided blocks)
        std::vector<int64_t> next_use(n, INT64_MAX);
        for (int64_t gi = (int64_t)rem_logical.size() - 1; gi >= 0; --gi) {
            const Gate& g = rem_logical[(size_t)gi];
            if (!is_diag(g)) next_use[g.t] = gi;
        }
        // victims sit at positions >= min_pos so each exchanged block is a set of
        // contiguous runs of >= 2^min_pos amplitudes (packed / unpacked at HBM speed)
        static const int min_pos_env = [] {
            const char* e = std::getenv("QG_REMAP_MIN_POS");
            return e ? std::atoi(e) : -1;
        }();
        const int min_pos = std::max(0, std::min(n_local - (int)need.size(),
                                                 min_pos_env >= 0 ? min_pos_env : kRemapMinPos));
        std::vector<int> cand;
        for (int pl = min_pos; pl < n_local; ++pl) cand.push_back(pl);
        std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) {
            const int64_t ua = next_use[inv[a]], ub = next_use[inv[b]];
            return ua != ub ? ua > ub : a > b;
        });
        std::vector<int> victims(cand.begin(), cand.begin() + rm.s);
        std::sort(victims.begin(), victims.end());
        for (int j = 0; j < rm.s; ++j) {
            rm.global_pos[j] = need[j];
            rm.local_pos[j] = victims[j];
        }
        for (int j = 0; j < rm.s; ++j) {
            const int pg = rm.global_pos[j], pl = rm.local_pos[j];
            const int lg = inv[pg], ll = inv[pl];
            std::swap(inv[pg], inv[pl]);
            phys[lg] = pl;
            phys[ll] = pg;
        }
        plan.remaps.push_back(rm);
        plan.segs.emplace_back();
    }
    plan.final_phys = phys;

    plan.body = body;
    return build_descriptors(plan, err);
    return QG_OK;
}

}  // namespace qg
