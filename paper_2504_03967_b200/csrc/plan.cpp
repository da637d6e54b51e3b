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
#include <cmath>
#include <complex>
#include <cstring>

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
        body.push_back(Gate{k, (k == K_CX || k == K_CR1) ? c : -1, t, p});
    }
    return QG_OK;
}

// ------------------------------------------------------------------ kernel configs
static const KernelCfg kCfgC64[] = {{0, 5, 3}, {1, 4, 2}, {2, 3, 0}};
static const KernelCfg kCfgC128[] = {{0, 4, 3}, {1, 3, 2}, {2, 3, 0}};

static bool pick_cfg(int dtype, int n_local, int force_k, KernelCfg& out) {
    const KernelCfg* cfgs = dtype == QG_DTYPE_C64 ? kCfgC64 : kCfgC128;
    if (force_k > 0) {
        for (int i = 0; i < 3; ++i)
            if (cfgs[i].k() == force_k && force_k <= n_local) { out = cfgs[i]; return true; }
        return false;
    }
    for (int i = 0; i < 3; ++i)
        if (n_local - cfgs[i].k() >= 8) { out = cfgs[i]; return true; }
    for (int i = 0; i < 3; ++i)
        if (cfgs[i].k() <= n_local) { out = cfgs[i]; return true; }
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

// per-amplitude instruction estimates; `in_reg` = register
// qubits of the stage being scanned (thread-level phases cost ~nothing per amp)
static double gate_cost(const Gate& g, const std::vector<char>& in_reg) {
    switch (g.kind) {
        case K_CX: return 1.5;
        case K_CR1: {
            const int r = (in_reg[g.c] ? 1 : 0) + (in_reg[g.t] ? 1 : 0);
            return r == 2 ? 1.0 : (r == 1 ? 2.0 : 0.1);
        }
        case K_RZ: return in_reg[g.t] ? 0.5 : 0.1;
        default: return 9.0;
    }
}
constexpr double kStageCost = 6.0;

struct StageSched {
    std::vector<int> regs;   // physical register qubits demanded (<= rb)
    std::vector<Gate> gates; // executed in this order (physical qubits)
};

// Schedules one fused pass from `rem` (physical-qubit gates, valid order);
// leaves the unscheduled gates in `rem` (still a valid order).
static void schedule_pass(std::vector<Gate>& rem, int n, int n_local, int k, int rb, int c_low, int max_stages,
                          double max_cost, std::vector<int>& tile, std::vector<StageSched>& stages) {
    std::vector<char> in_tile(n, 0);
    tile.clear();
    stages.clear();
    for (int q = 0; q < c_low && q < n_local; ++q) { in_tile[q] = 1; tile.push_back(q); }
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
                                 !(restrict_low && t < kLaneBits)) {
                            in_reg[t] = 1;
                            st.regs.push_back(t);
                            if (!in_tile[t]) { in_tile[t] = 1; tile.push_back(t); tile_added.push_back(t); }
                            ok = true;
                        }
                    }
                }
            }
            if (ok && cost + scost + gate_cost(g, in_reg) > max_cost && !st.gates.empty()) { ok = false; stop = true; }
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
        if (st.gates.empty()) {  // undo tile growth of an empty stage
            for (int q : tile_added) { in_tile[q] = 0; tile.erase(std::find(tile.begin(), tile.end(), q)); }
        }
    };
    for (int s = 0; s < max_stages && !rem.empty(); ++s) {
        StageSched st;
        std::vector<Gate> keep;
        double scost = 0;
        // stage 0 keeps the 5 lowest (lane) qubits out of registers so the tile
        // loads straight into the stage mapping; relax if that leaves it empty
        const bool restrict_low = s == 0 && c_low >= kLaneBits;
        scan(s, restrict_low, st, keep, scost);
        if (st.gates.empty() && restrict_low) {
            st = StageSched();
            scan(s, false, st, keep, scost);
        }
        if (st.gates.empty()) break;
        cost += scost;
        rem.swap(keep);
        stages.push_back(std::move(st));
        if (cost >= max_cost) break;
    }
    // fill the tile up to k qubits with the lowest unused local positions
    for (int q = 0; q < n_local && (int)tile.size() < k; ++q)
        if (!in_tile[q]) { in_tile[q] = 1; tile.push_back(q); }
    std::sort(tile.begin(), tile.end());
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
        for (int l = 0; l < kLaneBits; ++l) { hs.lane_tile.push_back(l); used[l] = 1; }
        for (int b = kLaneBits; b < k && (int)hs.reg_tile.size() < cfg.rb; ++b)
            if (!used[b]) { hs.reg_tile.push_back(b); used[b] = 1; }
    } else {
        for (int b = k - 1; b >= 0 && (int)hs.reg_tile.size() < cfg.rb; --b)
            if (!used[b]) { hs.reg_tile.push_back(b); used[b] = 1; }
        // conflict-free lanes: the lanes of one SMEM wavefront must cover every
        // residue class of the swizzle (8B amps: 16-lane phases, 4 classes mod 4;
        // 16B amps: 8-lane phases, 3 classes mod 3)
        const int M = dtype == QG_DTYPE_C64 ? 4 : 3;
        for (int r = 0; r < M; ++r)
            for (int b = 0; b < k; ++b)
                if (!used[b] && b % M == r) { hs.lane_tile.push_back(b); used[b] = 1; break; }
        for (int b = 0; b < k && (int)hs.lane_tile.size() < kLaneBits; ++b)
            if (!used[b]) { hs.lane_tile.push_back(b); used[b] = 1; }
    }
    for (int b = 0; b < k; ++b)
        if (!used[b]) { hs.warp_tile.push_back(b); used[b] = 1; }
}

static bool disjoint_low5(const std::vector<int>& bits) {
    for (int b : bits) if (b < kLaneBits) return false;
    return true;
}

// ------------------------------------------------------------------ op emission
struct Emitter {
    HostStage& hs;
    const std::vector<int>& tile_q;
    std::vector<int> reg_of;  // physical qubit -> register bit or -1
    std::vector<M2> pend;
    std::vector<char> has;
    Emitter(HostStage& h, const std::vector<int>& tq, int n) : hs(h), tile_q(tq), reg_of(n, -1) {
        for (size_t b = 0; b < hs.reg_tile.size(); ++b) reg_of[tile_q[hs.reg_tile[b]]] = (int)b;
        pend.resize(hs.reg_tile.size());
        has.assign(hs.reg_tile.size(), 0);
    }
    void op(int kind, int t, int c, int tq, int cq, uint64_t cmask, uint64_t qmask, const double* m, int nm) {
        HostOp o{};
        o.kind = kind; o.t = t; o.c = c; o.tq = tq; o.cq = cq; o.cmask = cmask; o.qmask = qmask;
        for (int i = 0; i < nm; ++i) o.m[i] = m[i];
        if (kind == OP_TPHASE) hs.tphase = true;
        hs.ops.push_back(o);
    }
    void flush(int b) {
        if (!has[b]) return;
        has[b] = 0;
        const M2& m = pend[b];
        const int q = tile_q[hs.reg_tile[b]];
        if (m.a01 == cd(0) && m.a10 == cd(0)) {
            if (m.a00 == cd(1) && m.a11 == cd(1)) return;
            if (m.a00 == cd(1)) {  // phase on |1> only; c = 1 marks "lo untouched"
                double d[4] = {1.0, 0.0, m.a11.real(), m.a11.imag()};
                op(OP_DIAG, b, 1, q, -1, 0, 0, d, 4);
                return;
            }
            double d[4] = {m.a00.real(), m.a00.imag(), m.a11.real(), m.a11.imag()};
            op(OP_DIAG, b, 0, q, -1, 0, 0, d, 4);
            return;
        }
        double d[8];
        put(d, m);
        op(OP_DENSE, b, -1, q, -1, 0, 0, d, 8);
    }
    void fold(int b, const M2& m) {
        pend[b] = has[b] ? mul(m, pend[b]) : m;
        has[b] = 1;
    }
    void gate(const Gate& g) {
        const int rt = reg_of[g.t];
        switch (g.kind) {
            case K_H: case K_RX: case K_RY:
                fold(rt, gate_matrix(g.kind, g.p));
                break;
            case K_RZ: {
                const M2 m = gate_matrix(K_RZ, g.p);
                if (rt >= 0) fold(rt, m);
                else {
                    double v[4] = {m.a00.real(), m.a00.imag(), m.a11.real(), m.a11.imag()};
                    op(OP_TPHASE, -1, -1, g.t, -1, 0, 1ull << g.t, v, 4);
                }
                break;
            }
            case K_CX: {
                flush(rt);
                const int rc = reg_of[g.c];
                if (rc >= 0) { flush(rc); op(OP_CX, rt, rc, g.t, g.c, 0, 0, nullptr, 0); }
                else op(OP_X, rt, -1, g.t, g.c, 1ull << g.c, 0, nullptr, 0);
                break;
            }
            case K_CR1: {
                const cd e = expi(g.p);
                const int rc = reg_of[g.c];
                if (rt >= 0 && rc >= 0) {
                    flush(rt); flush(rc);
                    double v[2] = {e.real(), e.imag()};
                    op(OP_CPHASE, std::max(rt, rc), std::min(rt, rc), g.t, g.c, 0, 0, v, 2);
                } else if (rt >= 0 || rc >= 0) {
                    const int b = rt >= 0 ? rt : rc;
                    const int other = rt >= 0 ? g.c : g.t;
                    flush(b);
                    double v[4] = {1.0, 0.0, e.real(), e.imag()};
                    op(OP_DIAG, b, 1, tile_q[hs.reg_tile[b]], other, 1ull << other, 0, v, 4);
                } else {
                    double v[4] = {e.real(), e.imag(), e.real(), e.imag()};
                    op(OP_TPHASE, -1, -1, g.t, g.c, (1ull << g.t) | (1ull << g.c), 0, v, 4);
                }
                break;
            }
            default: break;
        }
    }
    void finish() {
        for (size_t b = 0; b < has.size(); ++b) flush((int)b);
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
    for (int s = 0; s < S; ++s) {
        std::vector<int> need;
        for (int q : stages[s].regs) need.push_back(tbit[q]);
        const bool compat = disjoint_low5(need);
        const bool io = compat && (s == 0 || s == S - 1);
        assign_mapping(dtype, cfg, need, io, hp.stages[s]);
        Emitter em(hp.stages[s], hp.tile_q, n);
        for (const Gate& g : stages[s].gates) em.gate(g);
        em.finish();
        hp.n_gates += (int)stages[s].gates.size();
    }
    auto is_io = [](const HostStage& h) {
        for (int l = 0; l < kLaneBits; ++l) if (h.lane_tile[l] != l) return false;
        return true;
    };
    hp.load_direct = is_io(hp.stages[0]);
    hp.store_direct = is_io(hp.stages[S - 1]);
    assign_mapping(dtype, cfg, {}, true, hp.io);
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
template <typename Real>
static void fill_stage(int dtype, const HostPass& hp, const HostStage& h, StageDesc& d) {
    std::memset(&d, 0, sizeof(d));
    for (size_t b = 0; b < h.reg_tile.size(); ++b) {
        d.reg_q[b] = (uint8_t)hp.tile_q[h.reg_tile[b]];
        d.reg_s[b] = (uint16_t)swz(dtype, 1 << h.reg_tile[b]);
    }
    for (size_t b = 0; b < h.lane_tile.size(); ++b) {
        d.lane_q[b] = (uint8_t)hp.tile_q[h.lane_tile[b]];
        d.lane_s[b] = (uint16_t)swz(dtype, 1 << h.lane_tile[b]);
    }
    for (size_t b = 0; b < h.warp_tile.size(); ++b) {
        d.warp_q[b] = (uint8_t)hp.tile_q[h.warp_tile[b]];
        d.warp_s[b] = (uint16_t)swz(dtype, 1 << h.warp_tile[b]);
    }
    d.has_tphase = h.tphase ? 1 : 0;
}

template <typename Real>
static bool build_desc(int dtype, const HostPass& hp, int n_local, PassDesc<Real>& d, std::string& err) {
    std::memset(&d, 0, sizeof(d));
    d.n_stages = (int)hp.stages.size();
    d.k = hp.cfg.k();
    d.load_direct = hp.load_direct;
    d.store_direct = hp.store_direct;
    d.n_tiles = 1ull << (n_local - d.k);
    for (int i = 0; i < d.k; ++i) d.tile_q[i] = (uint8_t)hp.tile_q[i];
    fill_stage<Real>(dtype, hp, hp.io, d.stg[0]);
    int no = 0;
    for (int s = 0; s < d.n_stages; ++s) {
        const HostStage& h = hp.stages[s];
        StageDesc& sd = d.stg[1 + s];
        fill_stage<Real>(dtype, hp, h, sd);
        sd.op_begin = (uint16_t)no;
        for (const HostOp& o : h.ops) {
            if (no >= kMaxOps) { err = "pass exceeds kMaxOps"; return false; }
            OpDesc& od = d.ops[no];
            od.kind = (uint8_t)o.kind;
            od.t = (uint8_t)(o.t < 0 ? 0 : o.t);
            od.c = (uint8_t)(o.c < 0 ? 0 : o.c);
            od.mat = (uint32_t)no;
            od.cmask = o.cmask;
            od.qmask = o.qmask;
            for (int i = 0; i < 8; ++i) d.mats[no][i] = (Real)o.m[i];
            ++no;
        }
        sd.op_end = (uint16_t)no;
    }
    return true;
}

// ------------------------------------------------------------------ driver
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
    bool fused = opts.fuse != 0 && pick_cfg(opts.dtype, n_local, opts.tile_qubits, cfg);
    if (opts.fuse != 0 && opts.tile_qubits > 0 && !fused) {
        err = "tile_qubits not available for this dtype / size";
        return QG_E_INVALID_ARG;
    }
    plan.cfg = cfg;
    const int max_stages = opts.max_stages > 0 ? std::min(opts.max_stages, kMaxStages) : 4;
    const double max_cost = opts.max_cost > 0 ? (double)opts.max_cost : 96.0;
    const int c_low = n_local >= 20 ? kLaneBits : 0;  // small states live in L2: no coalescing constraint

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
                schedule_pass(rem, n, n_local, cfg.k(), cfg.rb, c_low, max_stages, max_cost, tile, stages);
                if (stages.empty()) break;
                plan.segs.back().push_back(make_fused_pass(opts.dtype, cfg, n, tile, stages));
            } else {
                const Gate& g = rem.front();
                if (!is_diag(g) && g.t >= n_local) break;
                plan.segs.back().push_back(make_unfused_pass(g, n_local));
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
            if ((int)need.size() == plan.g) break;
        }
        if (need.empty()) { err = "planner made no progress"; return QG_E_PROTOCOL; }
        qg_remap rm{};
        rm.s = (int)need.size();
        for (int j = 0; j < rm.s; ++j) {
            rm.global_pos[j] = need[j];
            rm.local_pos[j] = n_local - rm.s + j;
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

    // device descriptors
    plan.desc_index.resize(plan.segs.size());
    for (size_t s = 0; s < plan.segs.size(); ++s) {
        for (const HostPass& hp : plan.segs[s]) {
            int64_t idx = -1;
            if (hp.fused) {
                if (plan.dtype == QG_DTYPE_C64) {
                    plan.d32.emplace_back();
                    if (!build_desc<float>(plan.dtype, hp, n_local, plan.d32.back(), err)) return QG_E_INVALID_ARG;
                    idx = (int64_t)plan.d32.size() - 1;
                } else {
                    plan.d64.emplace_back();
                    if (!build_desc<double>(plan.dtype, hp, n_local, plan.d64.back(), err)) return QG_E_INVALID_ARG;
                    idx = (int64_t)plan.d64.size() - 1;
                }
                plan.stats.n_stages += (int64_t)hp.stages.size();
                for (const HostStage& h : hp.stages) plan.stats.n_ops += (int64_t)h.ops.size();
            } else {
                plan.stats.n_ops += 1;
            }
            plan.desc_index[s].push_back(idx);
        }
    }
    return QG_OK;
}

}  // namespace qg
