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
// must match launch_fused in fused.cu
static const KernelCfg kCfgC64[] = {{0, 4, 4}, {1, 4, 3}, {2, 4, 2}, {3, 3, 0}};
static const KernelCfg kCfgC128[] = {{0, 4, 3}, {1, 3, 2}, {2, 3, 0}};
static int n_cfgs(int dtype) { return dtype == QG_DTYPE_C64 ? 4 : 3; }

static bool pick_cfg(int dtype, int n_local, int force_k, KernelCfg& out) {
    const KernelCfg* cfgs = dtype == QG_DTYPE_C64 ? kCfgC64 : kCfgC128;
    const int nc = n_cfgs(dtype);
    if (force_k > 0) {
        for (int i = 0; i < nc; ++i)
            if (cfgs[i].k() == force_k && force_k <= n_local) { out = cfgs[i]; return true; }
        return false;
    }
    for (int i = 0; i < nc; ++i)
        if (n_local - cfgs[i].k() >= 8) { out = cfgs[i]; return true; }
    for (int i = 0; i < nc; ++i)
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

struct StageSched {
    std::vector<int> regs;   // physical register qubits demanded (<= rb)
    std::vector<Gate> gates; // executed in this order (physical qubits)
};

// Schedules one fused pass from `rem` (physical-qubit gates, valid order);
// leaves the unscheduled gates in `rem` (still a valid order).
static void schedule_pass(std::vector<Gate>& rem, int n, int n_local, int k, int rb, int c_low, int max_stages,
                          double max_cost, int max_gates, std::vector<int>& tile, std::vector<StageSched>& stages) {
    int n_taken = 0;
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
// Converts the stage's gates (program order) to register-level ops: consecutive
// 1-qubit gates on one register qubit are multiplied into one 2x2 in fp64 (real
// when possible); diagonal actions become predicated entries.
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
    static bool diagonal(const M2& m) { return m.a01 == cd(0) && m.a10 == cd(0); }
    HostOp mk(int kind, int t, int c, uint64_t cmask, uint64_t qmask) {
        HostOp o{};
        o.kind = kind; o.t = t; o.c = c;
        o.tq = t >= 0 ? tile_q[hs.reg_tile[t]] : -1;
        o.cq = c >= 0 ? tile_q[hs.reg_tile[c]] : -1;
        o.cmask = cmask; o.qmask = qmask;
        return o;
    }
    void flush(int b) {
        if (!has[b]) return;
        has[b] = 0;
        const M2& m = pend[b];
        if (diagonal(m)) {
            if (m.a00 == cd(1) && m.a11 == cd(1)) return;
            HostOp o = mk(A_CDIAG, b, -1, 0, 0);
            o.m[0] = m.a00.real(); o.m[1] = m.a00.imag(); o.m[2] = m.a11.real(); o.m[3] = m.a11.imag();
            hs.ops.push_back(o);
            return;
        }
        const bool real = m.a00.imag() == 0 && m.a01.imag() == 0 && m.a10.imag() == 0 && m.a11.imag() == 0;
        HostOp o = mk(real ? A_RDENSE : A_DENSE, b, -1, 0, 0);
        if (real) { o.m[0] = m.a00.real(); o.m[1] = m.a01.real(); o.m[2] = m.a10.real(); o.m[3] = m.a11.real(); }
        else put(o.m, m);
        hs.ops.push_back(o);
    }
    // an op acting diagonally on b: a pending diagonal commutes with it, a dense one must go first
    void flush_nondiag(int b) {
        if (has[b] && !diagonal(pend[b])) flush(b);
    }
    void fold(int b, const M2& m) {
        pend[b] = has[b] ? mul(m, pend[b]) : m;
        has[b] = 1;
    }
    void tph(uint64_t cmask, uint64_t qmask, cd v0, cd v1) {
        HostOp o = mk(A_TPH, -1, -1, cmask, qmask);
        o.m[0] = v0.real(); o.m[1] = v0.imag(); o.m[2] = v1.real(); o.m[3] = v1.imag();
        hs.tph.push_back(o);
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
                else tph(0, 1ull << g.t, m.a00, m.a11);
                break;
            }
            case K_CX: {
                flush(rt);
                const int rc = reg_of[g.c];
                if (rc >= 0) {
                    flush_nondiag(rc);
                    hs.ops.push_back(mk(A_CX, rt, rc, 0, 0));
                } else {
                    HostOp o = mk(A_X, rt, -1, 1ull << g.c, 0);
                    o.cq = g.c;
                    hs.ops.push_back(o);
                }
                break;
            }
            case K_CR1: {
                const cd e = expi(g.p);
                const int rc = reg_of[g.c];
                if (rt >= 0 && rc >= 0) {
                    flush_nondiag(rt);
                    flush_nondiag(rc);
                    HostOp o = mk(A_CP, std::max(rt, rc), std::min(rt, rc), 0, 0);
                    o.m[0] = e.real(); o.m[1] = e.imag();
                    hs.ops.push_back(o);
                } else if (rt >= 0 || rc >= 0) {
                    const int b = rt >= 0 ? rt : rc;
                    const int other = rt >= 0 ? g.c : g.t;
                    flush_nondiag(b);
                    HostOp o = mk(A_DIAG, b, -1, 1ull << other, 0);
                    o.cq = other;
                    o.m[0] = 1.0; o.m[1] = 0.0; o.m[2] = e.real(); o.m[3] = e.imag();
                    hs.ops.push_back(o);
                } else {
                    tph((1ull << g.t) | (1ull << g.c), 0, e, e);
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

// ------------------------------------------------------------------ round packing
// Slot execution order inside a round (must match fused.cu): dense(b) < cdiag(b) <
// diag(b) < X(b) < CX(t,c) < CPHASE(t>c); within a group by bit / pair index.
static int slot_key(const HostOp& o) {
    switch (o.kind) {
        case A_DENSE: case A_RDENSE: return 0 * 64 + o.t;
        case A_CDIAG: return 1 * 64 + o.t;
        case A_DIAG: return 2 * 64 + o.t;
        case A_X: return 3 * 64 + o.t;
        case A_CX: return 4 * 64 + 5 * o.t + o.c;
        default: return 5 * 64 + o.t * (o.t - 1) / 2 + o.c;  // A_CP, t > c
    }
}

// does op act non-diagonally on register bit b? (-1 = does not touch b)
static int acts(const HostOp& o, int b) {
    switch (o.kind) {
        case A_DENSE: case A_RDENSE: case A_X: return o.t == b ? 1 : -1;
        case A_DIAG: case A_CDIAG: return o.t == b ? 0 : -1;
        case A_CX: return o.t == b ? 1 : (o.c == b ? 0 : -1);
        case A_CP: return (o.t == b || o.c == b) ? 0 : -1;
        default: return -1;
    }
}

static bool commute(const HostOp& x, const HostOp& y, int rb) {
    for (int b = 0; b < rb; ++b) {
        const int ax = acts(x, b), ay = acts(y, b);
        if (ax >= 0 && ay >= 0 && (ax == 1 || ay == 1)) return false;
    }
    return true;
}

// Register CX gates that commute with every later op of the stage are moved past
// its end: their index map M (GF(2)-linear on register bits) is folded into the
// stage's output addressing (out_vec[b] = M^-1 e_b), so they cost nothing.
static void defer_trailing_cx(HostStage& hs, int rb) {
    std::vector<HostOp> kept, deferred_rev;
    for (int p = (int)hs.ops.size() - 1; p >= 0; --p) {
        const HostOp& x = hs.ops[p];
        bool ok = x.kind == A_CX;
        if (ok)
            for (const HostOp& y : kept)
                if (!commute(x, y, rb)) { ok = false; break; }
        if (ok) deferred_rev.push_back(x);
        else kept.push_back(x);
    }
    std::reverse(kept.begin(), kept.end());
    hs.ops.swap(kept);
    hs.deferred.assign(deferred_rev.rbegin(), deferred_rev.rend());  // program order
    hs.out_vec.assign(rb, 0);
    for (int b = 0; b < rb; ++b) {
        uint32_t v = 1u << b;
        for (const HostOp& c : hs.deferred)  // M^-1 = C_k ... C_1 : apply C_1 first
            if (v & (1u << c.c)) v ^= 1u << c.t;
        hs.out_vec[b] = v;
    }
}

static void pack_rounds(HostStage& hs, int rb) {
    struct Placed { const HostOp* op; int round; int key; };
    std::vector<Placed> placed;
    // slot occupancy per round: key -> index in round op list (list slots may repeat)
    std::vector<std::vector<int>> used;  // used[r] = keys occupied by single-op slots
    std::vector<std::vector<HostOp>> rops;
    for (const HostOp& x : hs.ops) {
        const int kx = slot_key(x);
        int lo = 0;
        for (const Placed& p : placed)
            if (!commute(x, *p.op, rb)) lo = std::max(lo, kx > p.key ? p.round : p.round + 1);
        const bool list_slot = x.kind == A_DIAG || x.kind == A_X;
        int r = lo;
        for (;; ++r) {
            if (r == (int)rops.size()) { rops.emplace_back(); used.emplace_back(); }
            if (list_slot) {
                // diag / X slot on bit t: a list; only the slot *type* must match
                bool clash = false;
                for (int k : used[r]) if (k == kx) clash = true;  // a single-op slot with this key? (never)
                if (!clash) break;
            } else {
                bool clash = false;
                for (int k : used[r]) if (k == kx) clash = true;
                if (!clash) break;
            }
        }
        if (!list_slot) used[r].push_back(kx);
        rops[r].push_back(x);
        placed.push_back(Placed{&x, r, kx});
    }
    hs.rounds.clear();
    for (auto& ops : rops) {
        std::stable_sort(ops.begin(), ops.end(),
                         [](const HostOp& a, const HostOp& b) { return slot_key(a) < slot_key(b); });
        hs.rounds.push_back(HostRound{ops});
    }
}

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
        defer_trailing_cx(hp.stages[s], cfg.rb);
        pack_rounds(hp.stages[s], cfg.rb);
        hp.n_gates += (int)stages[s].gates.size();
    }
    auto is_io = [](const HostStage& h) {
        for (int l = 0; l < kLaneBits; ++l) if (h.lane_tile[l] != l) return false;
        return true;
    };
    hp.load_direct = is_io(hp.stages[0]);
    hp.store_direct = is_io(hp.stages[S - 1]);
    assign_mapping(dtype, cfg, {}, true, hp.io);
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
    for (size_t b = 0; b < h.reg_tile.size(); ++b) {
        const uint32_t v = b < h.out_vec.size() ? h.out_vec[b] : (1u << b);
        int tidx = 0;
        uint64_t g = 0;
        for (size_t r = 0; r < h.reg_tile.size(); ++r)
            if (v & (1u << r)) {
                tidx |= 1 << h.reg_tile[r];
                g |= 1ull << hp.tile_q[h.reg_tile[r]];
            }
        d.out_s[b] = (uint16_t)swz(dtype, tidx);
        d.out_g[b] = g;
    }
}

template <typename Real>
static void put_entry(Entry<Real>& e, const HostOp& o) {
    e.cmask = o.cmask;
    e.qmask = o.qmask;
    for (int i = 0; i < 4; ++i) e.v[i] = (Real)o.m[i];
}

// resource needs of a pass (descriptor capacity is checked by the scheduler)
struct PassSize { int rounds = 0, coef = 0, ent = 0; };
static PassSize pass_size(const HostPass& hp) {
    PassSize z;
    for (const HostStage& h : hp.stages) {
        z.rounds += (int)h.rounds.size();
        z.ent += (int)h.tph.size();
        for (const HostRound& r : h.rounds)
            for (const HostOp& o : r.ops) {
                if (o.kind == A_DENSE || o.kind == A_RDENSE || o.kind == A_CP || o.kind == A_CDIAG) ++z.coef;
                if (o.kind == A_DIAG || o.kind == A_X) ++z.ent;
            }
    }
    return z;
}

static bool fits(const HostPass& hp) {
    const PassSize z = pass_size(hp);
    return z.rounds <= kMaxRounds && z.coef <= kMaxCoef && z.ent <= kMaxEnt;
}

template <typename Real>
static bool build_desc(int dtype, const HostPass& hp, int n_local, PassDesc<Real>& d, std::string& err) {
    std::memset(&d, 0, sizeof(d));
    if (!fits(hp)) { err = "pass exceeds descriptor capacity"; return false; }
    d.n_stages = (int)hp.stages.size();
    d.k = hp.cfg.k();
    d.load_direct = hp.load_direct;
    d.store_direct = hp.store_direct;
    d.n_tiles = 1ull << (n_local - d.k);
    for (int i = 0; i < d.k; ++i) d.tile_q[i] = (uint8_t)hp.tile_q[i];
    {
        int nc0 = 0;
        for (int q = 0; q < n_local; ++q)
            if (std::find(hp.tile_q.begin(), hp.tile_q.end(), q) == hp.tile_q.end()) d.comp_q[nc0++] = (uint8_t)q;
    }
    fill_stage(dtype, hp, hp.io, d.stg[0]);
    int nr = 0, nc = 0, ne = 0;
    for (int s = 0; s < d.n_stages; ++s) {
        const HostStage& h = hp.stages[s];
        StageDesc& sd = d.stg[1 + s];
        fill_stage(dtype, hp, h, sd);
        sd.tph_begin = (uint16_t)ne;
        for (const HostOp& o : h.tph) put_entry(d.ent[ne++], o);
        sd.tph_end = (uint16_t)ne;
        sd.round_begin = (uint16_t)nr;
        for (const HostRound& hr : h.rounds) {
            RoundDesc& R = d.rounds[nr++];
            R.coef = (uint16_t)nc;
            R.ent = (uint16_t)ne;
            // slot order: ops are sorted by slot key, so appending in order matches the kernel
            for (const HostOp& o : hr.ops) {
                switch (o.kind) {
                    case A_DENSE:
                        R.dense |= (uint8_t)(1u << o.t);
                        for (int i = 0; i < 8; ++i) d.coef[nc][i] = (Real)o.m[i];
                        ++nc;
                        break;
                    case A_RDENSE:
                        R.rdense |= (uint8_t)(1u << o.t);
                        for (int i = 0; i < 4; ++i) d.coef[nc][i] = (Real)o.m[i];
                        ++nc;
                        break;
                    case A_CDIAG:
                        R.cdiag |= (uint8_t)(1u << o.t);
                        for (int i = 0; i < 4; ++i) d.coef[nc][i] = (Real)o.m[i];
                        ++nc;
                        break;
                    case A_DIAG:
                        if (!(R.diag & (1u << o.t))) R.dhi |= (uint8_t)(1u << o.t);
                        if (!(o.m[0] == 1.0 && o.m[1] == 0.0)) R.dhi &= (uint8_t)~(1u << o.t);
                        R.diag |= (uint8_t)(1u << o.t);
                        R.dcnt[o.t]++;
                        put_entry(d.ent[ne++], o);
                        break;
                    case A_X:
                        R.xs |= (uint8_t)(1u << o.t);
                        R.xcnt[o.t]++;
                        put_entry(d.ent[ne++], o);
                        break;
                    case A_CX:
                        R.cx |= 1u << (5 * o.t + o.c);
                        break;
                    case A_CP:
                        R.cp |= (uint16_t)(1u << (o.t * (o.t - 1) / 2 + o.c));
                        d.coef[nc][0] = (Real)o.m[0];
                        d.coef[nc][1] = (Real)o.m[1];
                        ++nc;
                        break;
                }
            }
        }
        sd.round_end = (uint16_t)nr;
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
                int max_gates = kMaxEnt;  // shrunk below if the descriptor overflows
                HostPass hp;
                for (;;) {
                    std::vector<Gate> trial(rem);
                    schedule_pass(trial, n, n_local, cfg.k(), cfg.rb, c_low, max_stages, max_cost, max_gates,
                                  tile, stages);
                    if (stages.empty()) break;
                    hp = make_fused_pass(opts.dtype, cfg, n, tile, stages);
                    if (fits(hp) || max_gates <= 1) { rem.swap(trial); break; }
                    max_gates = std::max(1, hp.n_gates * 3 / 4);
                }
                if (stages.empty()) break;
                plan.segs.back().push_back(std::move(hp));
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
                for (const HostStage& h : hp.stages) {
                    plan.stats.n_ops += (int64_t)(h.ops.size() + h.tph.size());
                    plan.stats.n_rounds += (int64_t)h.rounds.size();
                }
            } else {
                plan.stats.n_ops += 1;
            }
            plan.desc_index[s].push_back(idx);
        }
    }
    return QG_OK;
}

}  // namespace qg
