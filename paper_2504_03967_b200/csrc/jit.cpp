// jit.cpp — straight-line PTX per fused pass (see jit.h).
//
// The emitted kernel is fused.cu's fused_pass_kernel<float, RB, WB, NBUF,
// false> specialised to one PassDesc: the same persistent tile loop, io
// mapping, SMEM transposes, op semantics (desc.h) and floating-point operation
// order, so its results are bit-identical to the interpreter's.  What the
// specialisation removes (per tile and thread, for a 32q random CX-block pass):
//   * the op-word fetch + jump-table dispatch of every op (~11 instructions
//     and a dependent LDC -> BRX chain each);
//   * run-time coefficient offsets: coefficients are constant-bank operands;
//   * flip-vector selects where the planner's program proves the thread's flip
//     bit is 0 (tracked statically per slot bit);
//   * OC_CXM register moves: a permutation of registers is a rename;
//   * X-gate / phase lists: unrolled, each predicate a constant bit position;
//   * Gray-code address walks: an SMEM / global address is a base register
//     plus an immediate, one base per distinct low part of the slot offsets.
#include "jit.h"

#include <nvPTXCompiler.h>

#include <sched.h>

#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <functional>
#include <map>
#include <tuple>
#include <unordered_map>
#include <sstream>

namespace qg {

std::atomic<int64_t> g_cache_hits{0};

namespace {

int par(uint64_t x) { return __builtin_parityll(x); }

std::string u64s(uint64_t v) {
    char b[24];
    std::snprintf(b, sizeof b, "0x%llx", (unsigned long long)v);
    return b;
}

template <typename Real>
struct Gen {
    using PD = PassDesc<Real>;
    // complex64: amplitudes are packed f32x2 (.b64), math in FFMA2 / FMUL2;
    // complex128: amplitudes are .b128 registers unpacked into f64 for DFMA math
    static constexpr bool D = sizeof(Real) == 8;
    static constexpr int ES = D ? 16 : 8, ESL = D ? 4 : 3;  // amplitude bytes / log2
    const PD& P;
    int RB, WB, NBUF, R, NT, k;
    std::ostringstream o;
    int nq = 0, nr = 0, nf = 0, np = 0, nl = 0, nx = 0, nd = 0;
    int amap[64];          // slot -> %a register index (register CX moves rename)
    uint32_t fposs = 0;    // slot bits of the flip vector F that may be 1
    // bit 0: tile loads as cp.async into the SMEM buffer, issued a tile ahead; 2048: one CTA per SM
    // (up to 255 registers); 4096: register double-buffered tiles (the next tile's loads are issued
    // into a second register bank when a tile starts; implies 2048); 8192: two transpose buffers
    int variant = 1;
    int tbuf = 0;          // transpose buffer of the next transpose (variant 8192)
    bool first_tr = true;  // first transpose of the tile
    int reads_left = 0;    // SMEM buffer reads left in the tile (async loads: the last one frees it)
    // producer/consumer mode (QG_JIT_PC): one CTA per SM = two consumer groups of NT threads
    // (each runs alternate tiles in registers, like two CTAs) + one producer warp that fills a
    // ring of kPcBufs SMEM tile buffers with cp.async (stage 1's input layout); per buffer a
    // "full" mbarrier (producer -> consumers) and an "empty" one (the group's last SMEM read)
    bool pc = false;
    static constexpr int kPcBufs = 3;
    size_t tab_mb = 0;     // mbarriers: full[kPcBufs], empty[kPcBufs]
    size_t off_coef, off_ph, off_tph;
    // smem layout
    size_t buf_bytes, tab_gb, tab_pf, tab_uph, tab_hp;
    static constexpr size_t kMapBytes = 576;  // 32 x u64 + 16 x u64 + 32 x u32 + 16 x u32
    // decode table: code -> (fam, T, C); fam 7 = CXM, 8 = XF, 9 = END
    struct Dec { int fam = -1, t = -1, c = -1; };
    std::vector<Dec> dec;

    Gen(const PD& p, int rb, int wb, int nbuf, int var) : P(p), RB(rb), WB(wb), NBUF(nbuf), variant(var) {
        if (D) variant &= (8 | 16 | 32 | 128 | 16384 | 32768 | 524288 | 4194304 | 33554432);  // c128: no probes of
                                                                                          // the c64 memory path
        R = 1 << RB;
        NT = 32 << WB;
        k = P.k;
        off_coef = offsetof(PD, coef);
        off_ph = offsetof(PD, ph);
        off_tph = offsetof(PD, tph);
        buf_bytes = (size_t)ES << k;
        tab_gb = tbufs(var) * NBUF * buf_bytes;           // per mapping: [lane g | warp g | lane s | warp s]
        tab_pf = tab_gb + (size_t)(P.n_stages + 1) * kMapBytes;  // [lane part | warp part] of the prefetch offset
        tab_uph = tab_pf + 384;                                   // tile-uniform phase slots (float2 each)
        tab_hp = tab_uph + ES * (size_t)kMaxUph;                  // hoisted per-thread phase slots
        for (int i = 0; i < R; ++i) amap[i] = i;
        dec.resize(oc_end(RB) + 1);
        for (int t = 0; t < RB; ++t) {
            dec[oc_std(F_RD, RB, t)] = {F_RD, t, -1};
            dec[oc_std(F_CD, RB, t)] = {F_CD, t, -1};
            dec[oc_std(F_PH, RB, t)] = {F_PH, t, -1};
            for (int c = 0; c < RB; ++c) {
                if (c == t) continue;
                dec[oc_pair(F_RDW, RB, t, c)] = {F_RDW, t, c};
                dec[oc_pair(F_RDV, RB, t, c)] = {F_RDV, t, c};
                if (c < t) {
                    dec[oc_tri(F_PHW, RB, t, c)] = {F_PHW, t, c};
                    dec[oc_tri(F_PH2, RB, t, c)] = {F_PH2, t, c};
                }
                dec[oc_cxm(RB, t, c)] = {7, t, c};
            }
        }
        dec[oc_xf(RB)] = {8, -1, -1};
        dec[oc_end(RB)] = {9, -1, -1};
    }
    // variant 33554432: phase ops whose factor lists are predicated on thread-constant
    // positions (the stage's lane / warp bits, rank bits) get those factors multiplied
    // once per launch into a per-thread SMEM slot (QFT rows: lists of up to n entries
    // otherwise re-evaluated every tile); the tile-id-predicated rest stays per tile
    static constexpr int kMaxHoist = 12, kMinHoisted = 4;
    std::map<int, int> hoist;  // op index -> slot
    std::vector<std::pair<int, int>> hoist_ops;  // (stage, op index) per slot
    bool thread_const(int s, uint32_t pos) const {
        const StageDesc& S = P.stg[s];
        for (int l = 0; l < kLaneBits; ++l) if (S.lane_q[l] == pos) return true;
        for (int w = 0; w < WB; ++w) if (S.warp_q[w] == pos) return true;
        for (int i = 0; i < k; ++i) if (P.tile_q[i] == pos) return false;
        const int n_comp = 63 - __builtin_clzll(P.n_tiles);
        for (int i = 0; i < n_comp; ++i) if (P.comp_q[i] == pos) return false;
        return true;  // a rank bit
    }
    void plan_hoist() {
        hoist.clear();
        hoist_ops.clear();
        if (!(variant & 33554432)) return;
        std::vector<std::tuple<int, int, int>> cand;  // (-count, stage, op)
        for (int s = 1; s <= P.n_stages; ++s)
            for (int oi = P.stg[s].op_begin;; ++oi) {
                const uint32_t w = P.ops[oi], code = w & 0xffu;
                if (code >= dec.size() || dec[code].fam < 0 || dec[code].fam == 9) break;
                if (dec[code].fam != F_PH && dec[code].fam != F_PHW) continue;
                const int n = (w >> 8) & 0x7f, b = w >> 16;
                int c = 0;
                for (int kk = 1; kk < n; ++kk) c += thread_const(s, P.ph[b + kk].pos) ? 1 : 0;
                if (c >= kMinHoisted) cand.emplace_back(-c, s, oi);
            }
        std::sort(cand.begin(), cand.end());
        for (const auto& t : cand) {
            if ((int)hoist_ops.size() == kMaxHoist) break;
            hoist[std::get<2>(t)] = (int)hoist_ops.size();
            hoist_ops.emplace_back(std::get<1>(t), std::get<2>(t));
        }
    }
    size_t hoist_bytes() const { return hoist_ops.size() * (size_t)NT * ES; }
    static bool pc_wanted() {
        static const bool v = std::getenv("QG_JIT_PC") && std::atoi(std::getenv("QG_JIT_PC")) > 0;
        return v;
    }
    bool pc_ok() const {
        return !D && NBUF == 1 && RB == 5 && WB == 3 && P.n_uph == 0 && P.n_stages >= 1 &&
               !(variant & (1 | 2 | 4 | 16 | 64 | 2048 | 4096 | 8192 | 262144 | 536870912 | 1073741824 | 8388608));  // 16: the
        // consumers' buffer release counts the transposes
    }
    void enable_pc() {
        pc = true;
        tab_mb = kPcBufs * buf_bytes;
        tab_gb = tab_mb + 64;
        tab_pf = tab_gb + (size_t)(P.n_stages + 1) * kMapBytes;
        tab_uph = tab_pf + 384;
        tab_hp = tab_uph + ES * (size_t)kMaxUph;
    }
    // after plan_hoist(): the producer/consumer form, when wanted, covered and within SMEM
    bool pc_use() const {
        return pc_wanted() && pc_ok() && pc_smem_bytes(P) + hoist_bytes() <= (size_t)225 * 1024;
    }
    static size_t pc_smem_bytes(const PD& P) {
        return kPcBufs * ((size_t)ES << P.k) + 64 + (size_t)(P.n_stages + 1) * kMapBytes + 384 + ES * (size_t)kMaxUph;
    }
    std::string bsync() const { return pc ? "bar.sync %gbar, " + std::to_string(NT) + ";" : "bar.sync 0;"; }
    // Scoped SMEM hand-over barriers.  Warp w of mapping m holds exactly the tile indices
    // whose warp-position bits (StageDesc::warp_q, in order) spell w; register CX maps and
    // flip vectors only permute register bits.  So a transpose from mapping ma to mb moves
    // data only between warps that agree on the warp bits ma and mb share at the same
    // index: none differ -> the warp exchanges with itself (bar.warp.sync), one differs
    // (WB = 3) -> pairs {w, w ^ 2^j} (named barrier 1 + 4j + the pair index, 64 threads;
    // one id per member set, so warps that drift apart never share an id across different
    // groups), otherwise the whole CTA.  Write-after-read inside a tile needs no CTA
    // barrier: a transpose's writers store the tile indices their own warp read in the
    // previous transpose (same mapping).
    bool wsync_ = false;
    int last_dst_ = -1;  // mapping of a tile's last SMEM read (the final transpose's target)
    std::string hand_sync(int ma, int mb) const {
        if (!wsync_) return bsync();
        const StageDesc &A = P.stg[ma], &B = P.stg[mb];
        int diff = 0, dj = -1;
        for (int j = 0; j < WB; ++j)
            if (A.warp_q[j] != B.warp_q[j]) { ++diff; dj = j; }
        if (std::getenv("QG_DEV_PLAN_DUMP")) std::fprintf(stderr, "handover %d -> %d: %d warp bits differ\n", ma, mb, diff);
        if (diff == 0) return "bar.warp.sync -1;";
        if (diff == 1 && WB == 3) return "bar.sync %gid" + std::to_string(dj) + ", 64;";
        return bsync();
    }
    // variant 8192: transposes alternate between two SMEM tile buffers (one barrier each)
    static int tbufs(int var) { return (var & 8192) ? 2 : 1; }
    static size_t smem_bytes(const PD& P, int rb, int wb, int nbuf, int var) {
        (void)rb;
        (void)wb;
        return tbufs(var) * nbuf * ((size_t)ES << P.k) + (size_t)(P.n_stages + 1) * kMapBytes + 384 +
               ES * (size_t)kMaxUph;
    }

    std::string q() { return "%q" + std::to_string(nq++); }
    std::string r() { return "%r" + std::to_string(nr++); }
    std::string f() { return "%f" + std::to_string(nf++); }
    std::string p() { return "%p" + std::to_string(np++); }
    std::string xq() { return "%x" + std::to_string(nx++); }  // .b128 (complex128 value)
    std::string dq() { return "%d" + std::to_string(nd++); }  // .f64
    std::string cv() { return D ? xq() : q(); }               // a complex value
    std::string sv() { return D ? dq() : f(); }               // a real scalar
    static constexpr const char* ST = D ? "f64" : "f32";
    static constexpr const char* ONE = D ? "0d3FF0000000000000" : "0f3F800000";
    static constexpr const char* ZERO = D ? "0d0000000000000000" : "0f00000000";
    static constexpr const char* CB = D ? "b128" : "b64";     // bit type of a complex value
    // parameter-space offsets of the Real-typed fields
    static size_t phe(int idx, int part) {  // PhEnt<Real> idx, part 0 = re, 1 = im
        return offsetof(PD, ph) + sizeof(PhEnt<Real>) * (size_t)idx + offsetof(PhEnt<Real>, e) + sizeof(Real) * part;
    }
    static size_t tphv(int idx, int kk) {   // Entry<Real> idx, v[kk]
        return offsetof(PD, tph) + sizeof(Entry<Real>) * (size_t)idx + offsetof(Entry<Real>, v) + sizeof(Real) * kk;
    }
    size_t coefo(uint32_t c) const { return off_coef + sizeof(Real) * (size_t)c; }
    std::string lab() { return "$J" + std::to_string(nl++); }
    // amplitude register of a slot: complex64 a packed .b64; complex128 a virtual name "%A<i>"
    // standing for the f64 pair (%ar<i>, %ai<i>) — unpack / pack_into resolve it without moves
    std::string a(int slot) const { return (D ? "%A" : "%a") + std::to_string(amap[slot]); }
    static bool is_amp(const std::string& c) { return D && c.size() > 2 && c[0] == '%' && c[1] == 'A'; }
    // memory-operand form of an amplitude register and the matching access type
    std::string amem(const std::string& c) const {
        return is_amp(c) ? "{%ar" + c.substr(2) + ", %ai" + c.substr(2) + "}" : c;
    }
    static constexpr const char* MT = D ? "v2.f64" : "b64";
    template <class... A>
    void L(const A&... x) {
        o << "\t";
        (o << ... << x);
        o << "\n";
    }

    // ---------------------------------------------------------------- values
    std::string ldp_f32(size_t off) {  // a Real scalar from the parameter space
        std::string v = sv();
        L("ld.param.", ST, " ", v, ", [P+", off, "];");
        return v;
    }
    std::string bc(const std::string& fv) {  // {v, v} (complex64); the scalar itself (complex128)
        if (D) return fv;
        std::string v = q();
        L("mov.b64 ", v, ", {", fv, ", ", fv, "};");
        return v;
    }
    std::pair<std::string, std::string> unpack(const std::string& c) {
        if (is_amp(c)) return {"%ar" + c.substr(2), "%ai" + c.substr(2)};
        std::string xr = sv(), xi = sv();
        L("mov.", CB, " {", xr, ", ", xi, "}, ", c, ";");
        return {xr, xi};
    }
    std::string shfl_s(const std::string& v, int o2) {  // butterfly shuffle of a Real scalar
        std::string out = sv();
        if (!D) {
            L("shfl.sync.bfly.b32 ", out, ", ", v, ", ", o2, ", 31, 0xffffffff;");
            return out;
        }
        std::string lo = r(), hi = r(), slo = r(), shi = r();
        L("mov.b64 {", lo, ", ", hi, "}, ", v, ";");
        L("shfl.sync.bfly.b32 ", slo, ", ", lo, ", ", o2, ", 31, 0xffffffff;");
        L("shfl.sync.bfly.b32 ", shi, ", ", hi, ", ", o2, ", 31, 0xffffffff;");
        L("mov.b64 ", out, ", {", slo, ", ", shi, "};");
        return out;
    }
    void pack_into(const std::string& d, const std::string& x, const std::string& y) {
        if (is_amp(d)) {
            L("mov.f64 %ar", d.substr(2), ", ", x, ";");
            L("mov.f64 %ai", d.substr(2), ", ", y, ";");
            return;
        }
        L("mov.", CB, " ", d, ", {", x, ", ", y, "};");
    }
    // complex value: a if pred else b
    std::string csel(const std::string& a_, const std::string& b_, const std::string& pred) {
        std::string v = cv();
        if (!D) {
            L("selp.b64 ", v, ", ", a_, ", ", b_, ", ", pred, ";");
            return v;
        }
        auto [ar, ai] = unpack(a_);
        auto [br, bi] = unpack(b_);
        std::string vr = dq(), vi = dq();
        L("selp.f64 ", vr, ", ", ar, ", ", br, ", ", pred, ";");
        L("selp.f64 ", vi, ", ", ai, ", ", bi, ", ", pred, ";");
        pack_into(v, vr, vi);
        return v;
    }
    // x += s * y (the shear of p_rot), in place
    void rfma(const std::string& x, const std::string& y, const std::string& s2) {
        if (!D) {
            L("fma.rn.f32x2 ", x, ", ", y, ", ", s2, ", ", x, ";");
            return;
        }
        auto [xr, xi] = unpack(x);
        auto [yr, yi] = unpack(y);
        std::string nr_ = dq(), ni_ = dq();
        L("fma.rn.f64 ", nr_, ", ", yr, ", ", s2, ", ", xr, ";");
        L("fma.rn.f64 ", ni_, ", ", yi, ", ", s2, ", ", xi, ";");
        pack_into(x, nr_, ni_);
    }
    // complex multiply / multiply-add in fused.cu's exact operation order
    std::string swp(const std::string& x) {  // {-x.y, x.x}
        std::string xr = f(), xi = f(), n = f(), s = q();
        L("mov.b64 {", xr, ", ", xi, "}, ", x, ";");
        L("neg.f32 ", n, ", ", xi, ";");
        L("mov.b64 ", s, ", {", n, ", ", xr, "};");
        return s;
    }
    void c_mul(const std::string& d, const std::string& x, const std::string& mr2, const std::string& mi2) {
        if (D) {  // d = x * (mr + i mi): (xr mr - xi mi, xi mr + xr mi)
            auto [xr, xi] = unpack(x);
            std::string tr = dq(), ti = dq(), nm = dq(), dr = dq(), di = dq();
            L("mul.rn.f64 ", tr, ", ", xr, ", ", mr2, ";");
            L("mul.rn.f64 ", ti, ", ", xi, ", ", mr2, ";");
            L("neg.f64 ", nm, ", ", mi2, ";");
            L("fma.rn.f64 ", dr, ", ", xi, ", ", nm, ", ", tr, ";");
            L("fma.rn.f64 ", di, ", ", xr, ", ", mi2, ", ", ti, ";");
            pack_into(d, dr, di);
            return;
        }
        std::string s = swp(x), t = q();
        L("mul.rn.f32x2 ", t, ", ", x, ", ", mr2, ";");
        L("fma.rn.f32x2 ", d, ", ", s, ", ", mi2, ", ", t, ";");
    }
    void c_fma(const std::string& d, const std::string& acc, const std::string& x, const std::string& mr2,
               const std::string& mi2) {
        if (D) {  // d = acc + x * (mr + i mi)
            auto [xr, xi] = unpack(x);
            auto [ar, ai] = unpack(acc);
            std::string tr = dq(), ti = dq(), nm = dq(), dr = dq(), di = dq();
            L("fma.rn.f64 ", tr, ", ", xr, ", ", mr2, ", ", ar, ";");
            L("fma.rn.f64 ", ti, ", ", xi, ", ", mr2, ", ", ai, ";");
            L("neg.f64 ", nm, ", ", mi2, ";");
            L("fma.rn.f64 ", dr, ", ", xi, ", ", nm, ", ", tr, ";");
            L("fma.rn.f64 ", di, ", ", xr, ", ", mi2, ", ", ti, ";");
            pack_into(d, dr, di);
            return;
        }
        std::string s = swp(x), t = q();
        L("fma.rn.f32x2 ", t, ", ", x, ", ", mr2, ", ", acc, ";");
        L("fma.rn.f32x2 ", d, ", ", s, ", ", mi2, ", ", t, ";");
    }
    // packed complex e -> ({e.x, e.x}, {e.y, e.y})
    std::pair<std::string, std::string> split_bc(const std::string& e) {
        auto [ex, ey] = unpack(e);
        return {bc(ex), bc(ey)};
    }
    std::string pack(const std::string& x, const std::string& y) {
        std::string v = cv();
        pack_into(v, x, y);
        return v;
    }
    // 1 if bit `pos` of the 64-bit value v is set (u32 0/1)
    std::string bit(const std::string& v64, int pos) {
        std::string t = q(), u = r();
        L("shr.b64 ", t, ", ", v64, ", ", pos, ";");
        L("cvt.u32.u64 ", u, ", ", t, ";");
        L("and.b32 ", u, ", ", u, ", 1;");
        return u;
    }
    std::string pred_nz(const std::string& u32) {
        std::string pp = p();
        L("setp.ne.u32 ", pp, ", ", u32, ", 0;");
        return pp;
    }
    // parity(W & F) as a predicate (F runtime)
    std::string fpar(uint32_t W) {
        std::string t = r(), pp = p();
        L("and.b32 ", t, ", %F, ", W, ";");
        L("popc.b32 ", t, ", ", t, ";");
        L("and.b32 ", t, ", ", t, ", 1;");
        L("setp.ne.u32 ", pp, ", ", t, ", 0;");
        return pp;
    }

    // ---------------------------------------------------------------- ops
    // rotation as three in-place shears on pairs {i, i ^ V}, x = parity(W & i) = 0 member
    // slot filter (variant 4194304): emit only slots with (slot & fmask) == fval
    uint32_t fmask = 0, fval = 0;
    bool in_sub(int i) const { return ((uint32_t)i & fmask) == fval; }
    void p_rot(uint32_t V, uint32_t W, const std::string& sa2, const std::string& sb2) {
        for (int pass = 0; pass < 3; ++pass)
            for (int i = 0; i < R; ++i) {
                if (par(W & (uint32_t)i) || !in_sub(i)) continue;
                const int j = i ^ (int)V;
                if (pass == 1) rfma(a(j), a(i), sb2);
                else rfma(a(i), a(j), sa2);
            }
    }
    // packed complex64 negation (ptxas folds it into the consuming FFMA2's operand)
    std::string negc(const std::string& v) {
        auto [xr, xi] = unpack(v);
        std::string nr = sv(), ni = sv();
        L("neg.f32 ", nr, ", ", xr, ";");
        L("neg.f32 ", ni, ", ", xi, ";");
        return pack(nr, ni);
    }
    // complex64 rotation in the planner's scaled form (plan.cpp Emitter::rotation), the same
    // fmas as fused.cu p_rot_scaled: form 0 x' = x - k y, y' = y + k x; form 1 x' = k x - y,
    // y' = x + k y; swapped roles (flip vector) see -k / the unit terms negated
    void op_rd_scaled(uint32_t V, uint32_t W, uint32_t coef) {
        const bool form1 = P.coef[coef + 1] != 0;
        const std::string k = ldp_f32(coefo(coef));
        const bool fl = (W & fposs) != 0;
        const std::string fp = fl ? fpar(W) : std::string();
        if (!form1) {
            std::string kk = k;
            if (fl) {
                std::string nk0 = sv();
                kk = sv();
                L("neg.f32 ", nk0, ", ", k, ";");
                L("selp.f32 ", kk, ", ", nk0, ", ", k, ", ", fp, ";");
            }
            std::string nkk = sv();
            L("neg.f32 ", nkk, ", ", kk, ";");
            const std::string kk2 = bc(kk), nkk2 = bc(nkk);
            for (int i = 0; i < R; ++i) {
                if (par(W & (uint32_t)i) || !in_sub(i)) continue;
                const int j = i ^ (int)V;
                std::string t = q();
                L("fma.rn.f32x2 ", t, ", ", a(j), ", ", nkk2, ", ", a(i), ";");
                L("fma.rn.f32x2 ", a(j), ", ", a(i), ", ", kk2, ", ", a(j), ";");
                L("mov.b64 ", a(i), ", ", t, ";");
            }
            return;
        }
        const std::string k2 = bc(k);
        for (int i = 0; i < R; ++i) {
            if (par(W & (uint32_t)i) || !in_sub(i)) continue;
            const int j = i ^ (int)V;
            const std::string ny = negc(a(j));
            std::string ax = ny, ay = a(i);
            if (fl) {
                ax = csel(a(j), ny, fp);           // flipped: + y
                ay = csel(negc(a(i)), a(i), fp);   // flipped: - x
            }
            std::string t = q();
            L("fma.rn.f32x2 ", t, ", ", a(i), ", ", k2, ", ", ax, ";");
            L("fma.rn.f32x2 ", a(j), ", ", a(j), ", ", k2, ", ", ay, ";");
            L("mov.b64 ", a(i), ", ", t, ";");
        }
    }
    void op_rd(uint32_t V, uint32_t W, uint32_t coef) {
        if (!D) {
            op_rd_scaled(V, W, coef);
            return;
        }
        std::string m0 = ldp_f32(coefo(coef)), m1 = ldp_f32(coefo(coef + 1));
        std::string sa = m0, sb = m1;
        if (W & fposs) {
            std::string fp = fpar(W), n0 = sv(), n1 = sv();
            sa = sv();
            sb = sv();
            L("neg.", ST, " ", n0, ", ", m0, ";");
            L("neg.", ST, " ", n1, ", ", m1, ";");
            L("selp.", ST, " ", sa, ", ", n0, ", ", m0, ", ", fp, ";");
            L("selp.", ST, " ", sb, ", ", n1, ", ", m1, ", ", fp, ";");
        }
        p_rot(V, W, bc(sa), bc(sb));
    }
    void op_cd(uint32_t V, uint32_t W, uint32_t coef) {
        std::string m[8];
        for (int i = 0; i < 8; ++i) m[i] = ldp_f32(coefo(coef + i));
        std::string c[8];
        if (W & fposs) {  // X U X: c = (m11, m10, m01, m00)
            std::string fp = fpar(W);
            static const int sw[8] = {6, 7, 4, 5, 2, 3, 0, 1};
            for (int i = 0; i < 8; ++i) {
                c[i] = sv();
                L("selp.", ST, " ", c[i], ", ", m[sw[i]], ", ", m[i], ", ", fp, ";");
            }
        } else {
            for (int i = 0; i < 8; ++i) c[i] = m[i];
        }
        std::string c00r = bc(c[0]), c00i = bc(c[1]), c01r = bc(c[2]), c01i = bc(c[3]);
        std::string c10r = bc(c[4]), c10i = bc(c[5]), c11r = bc(c[6]), c11i = bc(c[7]);
        for (int i = 0; i < R; ++i) {
            if (par(W & (uint32_t)i) || !in_sub(i)) continue;
            const int j = i ^ (int)V;
            std::string ty = cv(), tx = cv();
            c_mul(ty, a(j), c01r, c01i);
            c_mul(tx, a(i), c10r, c10i);
            c_fma(a(i), ty, a(i), c00r, c00i);
            c_fma(a(j), tx, a(j), c11r, c11i);
        }
    }
    // multiply slots with parity(W & i) == P by e (packed)
    void p_phase(uint32_t W, int Pp, const std::string& er2, const std::string& ei2) {
        for (int i = 0; i < R; ++i)
            if (par(W & (uint32_t)i) == Pp && in_sub(i)) c_mul(a(i), a(i), er2, ei2);
    }
    void op_ph(uint32_t W, const std::string& e) {
        auto [er2, ei2] = split_bc(e);
        if (!(W & fposs)) {
            p_phase(W, 1, er2, ei2);
            return;
        }
        std::string fp = fpar(W), bal = r(), p0 = p(), p1 = p();
        std::string la = lab(), lb = lab(), le = lab();
        L("vote.sync.ballot.b32 ", bal, ", ", fp, ", 0xffffffff;");
        L("setp.eq.u32 ", p0, ", ", bal, ", 0;");
        L("setp.eq.u32 ", p1, ", ", bal, ", 0xffffffff;");
        L("@", p0, " bra.uni ", la, ";");
        L("@", p1, " bra.uni ", lb, ";");
        {  // mixed warp: per-thread diag(d0, d1)
            auto [ex, ey] = unpack(e);
            std::string d0x = sv(), d0y = sv(), d1x = sv(), d1y = sv();
            L("selp.", ST, " ", d0x, ", ", ex, ", ", ONE, ", ", fp, ";");
            L("selp.", ST, " ", d0y, ", ", ey, ", ", ZERO, ", ", fp, ";");
            L("selp.", ST, " ", d1x, ", ", ONE, ", ", ex, ", ", fp, ";");
            L("selp.", ST, " ", d1y, ", ", ZERO, ", ", ey, ", ", fp, ";");
            std::string d0r = bc(d0x), d0i = bc(d0y), d1r = bc(d1x), d1i = bc(d1y);
            for (int i = 0; i < R; ++i) {
                if (!in_sub(i)) continue;
                if (par(W & (uint32_t)i)) c_mul(a(i), a(i), d1r, d1i);
                else c_mul(a(i), a(i), d0r, d0i);
            }
            L("bra.uni ", le, ";");
        }
        o << la << ":\n";
        p_phase(W, 1, er2, ei2);
        L("bra.uni ", le, ";");
        o << lb << ":\n";
        p_phase(W, 0, er2, ei2);
        o << le << ":\n";
    }
    // ph_product<false>: entry 0 unconditional, then predicated factors in list order
    bool prologue_ = false;
    // entry 0 times the thread-constant factors of op oi (stage s), tb = thread bits | rank bits
    std::string hoisted_product(int s, uint32_t w, const std::string& tb) {
        const int n = (w >> 8) & 0x7f, b = w >> 16;
        std::string ex = ldp_f32(phe(b, 0)), ey = ldp_f32(phe(b, 1));
        std::string e = pack(ex, ey);
        for (int kk = 1; kk < n; ++kk) {
            const PhEnt<Real>& E = P.ph[b + kk];
            if (!thread_const(s, E.pos)) continue;
            std::string on = pred_nz(bit(tb, (int)E.pos));
            std::string vx = sv(), vy = sv();
            std::string e0 = ldp_f32(phe(b + kk, 0)), e1 = ldp_f32(phe(b + kk, 1));
            L("selp.", ST, " ", vx, ", ", e0, ", ", ONE, ", ", on, ";");
            L("selp.", ST, " ", vy, ", ", e1, ", ", ZERO, ", ", on, ";");
            std::string ne = cv();
            c_mul(ne, e, bc(vx), bc(vy));
            e = ne;
        }
        return e;
    }
    int cur_op = -1, cur_stage = -1;  // the op / stage being emitted (hoisted phase slots)
    std::string ph_product(uint32_t w, const std::string& tb) {
        const int n = (w >> 8) & 0x7f, b = w >> 16;
        auto hz = hoist.find(cur_op);
        if (hz != hoist.end() && !prologue_) {  // entry 0 and the thread-constant factors: one LDS
            std::string e = cv();
            L("ld.shared.", CB, " ", e, ", [%hpb+", (size_t)hz->second * NT * ES, "];");
            if ((w & 0x8000u) && P.n_uph > 0) {
                std::string u = cv(), ne = cv(), ad = r();
                L("add.u32 ", ad, ", %smb, ", tab_uph + ES * (size_t)P.ph[b].pad, ";");
                L("ld.shared.", CB, " ", u, ", [", ad, "];");
                auto [ur2, ui2] = split_bc(u);
                c_mul(ne, e, ur2, ui2);
                e = ne;
            }
            for (int kk = 1; kk < n; ++kk) {
                const PhEnt<Real>& E = P.ph[b + kk];
                if (thread_const(cur_stage, E.pos)) continue;
                std::string on = pred_nz(bit(tb, (int)E.pos));
                std::string vx = sv(), vy = sv();
                std::string e0 = ldp_f32(phe(b + kk, 0)), e1 = ldp_f32(phe(b + kk, 1));
                L("selp.", ST, " ", vx, ", ", e0, ", ", ONE, ", ", on, ";");
                L("selp.", ST, " ", vy, ", ", e1, ", ", ZERO, ", ", on, ";");
                std::string ne = cv();
                c_mul(ne, e, bc(vx), bc(vy));
                e = ne;
            }
            return e;
        }
        std::string ex = ldp_f32(phe(b, 0)), ey = ldp_f32(phe(b, 1));
        std::string e = pack(ex, ey);
        if ((w & 0x8000u) && P.n_uph > 0) {  // the tile-uniform factors (computed at the tile start)
            std::string u = cv(), ne = cv(), ad = r();
            L("add.u32 ", ad, ", %smb, ", tab_uph + ES * (size_t)P.ph[b].pad, ";");
            L("ld.shared.", CB, " ", u, ", [", ad, "];");
            auto [ur2, ui2] = split_bc(u);
            c_mul(ne, e, ur2, ui2);
            e = ne;
        }
        for (int kk = 1; kk < n; ++kk) {
            const PhEnt<Real>& E = P.ph[b + kk];
            std::string on = pred_nz(bit(tb, (int)E.pos));
            std::string vx = sv(), vy = sv();
            std::string e0 = ldp_f32(phe(b + kk, 0)), e1 = ldp_f32(phe(b + kk, 1));
            L("selp.", ST, " ", vx, ", ", e0, ", ", ONE, ", ", on, ";");
            L("selp.", ST, " ", vy, ", ", e1, ", ", ZERO, ", ", on, ";");
            std::string ne = cv();
            c_mul(ne, e, bc(vx), bc(vy));
            e = ne;
        }
        return e;
    }
    void op_ph2(int T, int C, uint32_t coef) {
        std::string ex = ldp_f32(coefo(coef)), ey = ldp_f32(coefo(coef + 1));
        std::string er2 = bc(ex), ei2 = bc(ey);
        auto cphase = [&]() {
            for (int i = 0; i < R; ++i)
                if (((i >> T) & 1) && ((i >> C) & 1) && in_sub(i)) c_mul(a(i), a(i), er2, ei2);
        };
        if (!(fposs & ((1u << T) | (1u << C)))) {
            cphase();
            return;
        }
        std::string ft = r(), fc = r(), any = r(), bal = r(), p0 = p();
        L("bfe.u32 ", ft, ", %F, ", T, ", 1;");
        L("bfe.u32 ", fc, ", %F, ", C, ", 1;");
        L("or.b32 ", any, ", ", ft, ", ", fc, ";");
        std::string pany = pred_nz(any);
        L("vote.sync.ballot.b32 ", bal, ", ", pany, ", 0xffffffff;");
        L("setp.eq.u32 ", p0, ", ", bal, ", 0;");
        std::string la = lab(), le = lab();
        L("@", p0, " bra.uni ", la, ";");
        {  // r_cphase_flip: v = (bt & bc) ? e : 1 for every slot
            std::string vr[4], vi[4];
            for (int combo = 0; combo < 4; ++combo) {  // (slot bit T, slot bit C)
                const int st = combo & 1, sc = combo >> 1;
                std::string bt = r(), bcv = r(), both = r(), pp;
                L("xor.b32 ", bt, ", ", ft, ", ", st, ";");
                L("xor.b32 ", bcv, ", ", fc, ", ", sc, ";");
                L("and.b32 ", both, ", ", bt, ", ", bcv, ";");
                pp = pred_nz(both);
                std::string x = sv(), y = sv();
                L("selp.", ST, " ", x, ", ", ex, ", ", ONE, ", ", pp, ";");
                L("selp.", ST, " ", y, ", ", ey, ", ", ZERO, ", ", pp, ";");
                vr[combo] = bc(x);
                vi[combo] = bc(y);
            }
            for (int i = 0; i < R; ++i) {
                if (!in_sub(i)) continue;
                const int combo = ((i >> T) & 1) | (((i >> C) & 1) << 1);
                c_mul(a(i), a(i), vr[combo], vi[combo]);
            }
            L("bra.uni ", le, ";");
        }
        o << la << ":\n";
        cphase();
        o << le << ":\n";
    }
    void op_xf(uint32_t w, const std::string& tb) {
        const int n = (w >> 8) & 0xff, b = w >> 16;
        for (int kk = 0; kk < n; ++kk) {
            const uint32_t e = P.xfe[b + kk];
            const uint32_t v = e >> 8;
            std::string on = bit(tb, (int)(e & 63u)), m = r();
            L("neg.s32 ", m, ", ", on, ";");
            L("and.b32 ", m, ", ", m, ", ", v, ";");
            L("xor.b32 %F, %F, ", m, ";");
            fposs |= v;
        }
    }
    void op_cxm(int T, int C) {
        // r_cx: swap slots i and i | 1<<T for i with bit C set and bit T clear — a rename
        for (int i = 0; i < R; ++i) {
            if ((i & (1 << T)) || !(i & (1 << C))) continue;
            std::swap(amap[i], amap[i | (1 << T)]);
        }
        if (fposs & (1u << C)) {
            std::string t = r();
            L("bfe.u32 ", t, ", %F, ", C, ", 1;");
            L("shl.b32 ", t, ", ", t, ", ", T, ";");
            L("xor.b32 %F, %F, ", t, ";");
            fposs |= 1u << T;
        }
    }

    // ---------------------------------------------------------------- addressing
    // per-thread table entries (SMEM, written in the prologue)
    std::string gb_of(int m) {
        if (variant & 524288) {  // per-thread mapping values held in registers (no SMEM table reads)
            std::string v = q();
            L("mov.b64 ", v, ", %gbm", m, ";");
            return v;
        }
        std::string a1 = q(), a2 = q(), v = q();
        L("ld.shared.u64 ", a1, ", [%tl8+", (size_t)m * kMapBytes, "];");
        L("ld.shared.u64 ", a2, ", [%tw8+", (size_t)m * kMapBytes + 256, "];");
        L("or.b64 ", v, ", ", a1, ", ", a2, ";");
        return v;
    }
    std::string so_of(int m) {
        if (variant & 524288) {
            std::string v = r();
            L("mov.b32 ", v, ", %som", m, ";");
            return v;
        }
        std::string a1 = r(), a2 = r(), v = r();
        L("ld.shared.u32 ", a1, ", [%tl4+", (size_t)m * kMapBytes + 384, "];");
        L("ld.shared.u32 ", a2, ", [%tw4+", (size_t)m * kMapBytes + 512, "];");
        L("xor.b32 ", v, ", ", a1, ", ", a2, ";");
        return v;
    }
    // thread-bit masks of a mapping: global positions of lane/warp bits, SMEM byte-offset bits
    uint64_t thread_gmask(int m) const {
        uint64_t g = 0;
        for (int l = 0; l < kLaneBits; ++l) g |= 1ull << P.stg[m].lane_q[l];
        for (int w = 0; w < WB; ++w) g |= 1ull << P.stg[m].warp_q[w];
        return g;
    }
    uint32_t thread_smask(int m) const {
        uint32_t s = 0;
        for (int l = 0; l < kLaneBits; ++l) s |= (uint32_t)P.stg[m].lane_s[l] << ESL;
        for (int w = 0; w < WB; ++w) s |= (uint32_t)P.stg[m].warp_s[w] << ESL;
        return s;
    }
    // 64-bit value with large constant added, reusing bases per high part
    struct Bases {
        std::map<uint64_t, std::string> m;
    };
    std::string addr64(Bases& B, const std::string& base, uint64_t off) {
        const uint64_t hi = off >> 22, lo = off & ((1ull << 22) - 1);
        auto it = B.m.find(hi);
        std::string br;
        if (it == B.m.end()) {
            if (hi == 0) br = base;
            else {
                br = q();
                L("add.s64 ", br, ", ", base, ", ", u64s(hi << 22), ";");
            }
            B.m[hi] = br;
        } else {
            br = it->second;
        }
        return "[" + br + "+" + u64s(lo) + "]";
    }

    // SMEM store of every slot i at (T ^ O(i)), T runtime with bits within `lm`
    void smem_store(const std::string& T, uint32_t lm, const std::vector<uint32_t>& O,
                    const std::string& sb = "%smb") {
        std::map<uint32_t, std::string> base;
        for (int i = 0; i < R; ++i) {
            const uint32_t lo = O[i] & lm, hi = O[i] & ~lm;
            auto it = base.find(lo);
            std::string br;
            if (it == base.end()) {
                br = r();
                L("xor.b32 ", br, ", ", T, ", ", lo, ";");
                L("add.u32 ", br, ", ", br, ", ", sb, ";");
                base[lo] = br;
            } else {
                br = it->second;
            }
            L("st.shared.", MT, " [", br, "+", hi, "], ", amem(a(i)), ";");
        }
    }
    void smem_load(const std::string& T, uint32_t lm, const std::vector<uint32_t>& O,
                   const std::string& sb = "%smb") {
        std::map<uint32_t, std::string> base;
        for (int i = 0; i < R; ++i) {
            const uint32_t lo = O[i] & lm, hi = O[i] & ~lm;
            auto it = base.find(lo);
            std::string br;
            if (it == base.end()) {
                br = r();
                L("xor.b32 ", br, ", ", T, ", ", lo, ";");
                L("add.u32 ", br, ", ", br, ", ", sb, ";");
                base[lo] = br;
            } else {
                br = it->second;
            }
            L("ld.shared.", MT, " ", amem(a(i)), ", [", br, "+", hi, "];");
        }
    }

    // transpose from mapping m1 (with the current F) into mapping m2
    void transpose(int m1, int m2) {
        const bool two = (variant & 8192) != 0;
        if ((variant & 262144) && first_tr) L("cp.async.bulk.wait_group.read 0;");  // the last tile's stores
        // (variant 67108864: timing probe, warp-scoped barriers only — wrong results; bounds
        // what decoupling the warps of a CTA at the transposes could gain)
        const bool probe = (variant & 67108864) != 0;
        if (NBUF == 1 && (!two || first_tr)) {  // WAR on the buffer last read
            if (probe) L("bar.warp.sync -1;");
            else if (!wsync_) L(bsync());
            else L(first_tr ? hand_sync(last_dst_, m1) : std::string("bar.warp.sync -1;"));
        }
        first_tr = false;
        const std::string sb = pc ? std::string("%smc") : (two && tbuf) ? std::string("%smb2") : std::string("%smb");
        if (two) tbuf ^= 1;
        const StageDesc& S1 = P.stg[m1];
        std::string T = so_of(m1);
        uint32_t lm = thread_smask(m1);
        for (int b = 0; b < RB; ++b) {
            if (!(fposs & (1u << b))) continue;
            std::string t = r();
            L("bfe.u32 ", t, ", %F, ", b, ", 1;");
            L("neg.s32 ", t, ", ", t, ";");
            L("and.b32 ", t, ", ", t, ", ", S1.out_s[b], ";");
            L("xor.b32 ", T, ", ", T, ", ", t, ";");
            lm |= S1.out_s[b];
        }
        std::vector<uint32_t> O(R);
        for (int i = 0; i < R; ++i) {
            uint32_t v = 0;
            for (int b = 0; b < RB; ++b)
                if (i & (1 << b)) v ^= S1.out_s[b];
            O[i] = v;
        }
        smem_store(T, lm, O, sb);
        L(probe ? std::string("bar.warp.sync -1;") : hand_sync(m1, m2));
        for (int i = 0; i < R; ++i) amap[i] = i;  // register renames end with the stage
        const StageDesc& S2 = P.stg[m2];
        std::string T2 = so_of(m2);
        for (int i = 0; i < R; ++i) {
            uint32_t v = 0;
            for (int b = 0; b < RB; ++b)
                if (i & (1 << b)) v ^= S2.reg_s[b];
            O[i] = v;
        }
        smem_load(T2, thread_smask(m2), O, sb);
        L("mov.u32 %F, 0;");
        fposs = 0;
        after_read();
    }

    // the planner's SMEM swizzle of a tile index (plan.cpp swz, complex64); an involution
    static uint32_t swz(uint32_t j) { return j ^ (((j >> 4) ^ (j >> 8) ^ (j >> 12)) & 15u); }
    int run_bits() const {  // contiguous low qubits of the tile: one run = 2^c amplitudes in HBM
        int c = 0;
        while (c < k && P.tile_q[c] == c) ++c;
        return c;
    }
    // variant 262144: the tile leaves through the TMA engine.  The registers (store
    // mapping si, flips folded in) go to the SMEM buffer in the LINEAR tile-index layout
    // (offset = tile index * 8: each HBM run is one contiguous SMEM range), then warp 0
    // issues one cp.async.bulk shared -> global copy per run; the buffer is reused only
    // after the copies have read it (cp.async.bulk.wait_group.read before the tile's
    // first SMEM write).  Warps never wait on the stores' L2 / HBM write path.
    void tma_store(int si) {
        const StageDesc& S = P.stg[si];
        L("cp.async.bulk.wait_group.read 0;");
        L("bar.sync 0;");  // WAR: the buffer's last reads (final transpose) are done
        std::string T = r();
        L("mov.u32 ", T, ", %tlin;");
        uint32_t lm = tlin_mask;
        uint32_t Ol[kMaxRegBits];
        for (int b = 0; b < RB; ++b) Ol[b] = swz(S.out_s[b] >> 3) << 3;
        for (int b = 0; b < RB; ++b) {
            if (!(fposs & (1u << b))) continue;
            std::string t = r();
            L("bfe.u32 ", t, ", %F, ", b, ", 1;");
            L("neg.s32 ", t, ", ", t, ";");
            L("and.b32 ", t, ", ", t, ", ", Ol[b], ";");
            L("xor.b32 ", T, ", ", T, ", ", t, ";");
            lm |= Ol[b];
        }
        std::vector<uint32_t> O(R);
        for (int i = 0; i < R; ++i) {
            uint32_t v = 0;
            for (int b = 0; b < RB; ++b)
                if (i & (1 << b)) v ^= Ol[b];
            O[i] = v;
        }
        smem_store(T, lm, O, "%smb");
        L("fence.proxy.async.shared::cta;");
        L("bar.sync 0;");
        const int c = run_bits(), nrb = k - c;  // 2^nrb runs of 2^c amplitudes
        const int64_t nr = 1ll << nrb, rs = 8ll << c;
        std::string ls = lab();
        L("@!%pw0 bra.uni ", ls, ";");
        std::string pl = p();
        if (nr < 32) {
            L("setp.ge.u32 ", pl, ", %xlane, ", nr, ";");
            L("@", pl, " bra.uni ", ls, ";");
        }
        std::string gl = q(), sl = r();
        L("or.b64 ", gl, ", %base, %rdl;");    // tile base | this lane's run bits (deposited)
        L("shl.b32 ", sl, ", %xlane, ", c + 3, ";");
        L("add.u32 ", sl, ", ", sl, ", %smb;");
        for (int64_t m = 0; m * 32 < nr; ++m) {
            uint64_t dm = 0;  // run bits 5.. of run index 32 m
            for (int i = 5; i < nrb; ++i)
                if (((32 * m) >> i) & 1) dm |= 1ull << P.tile_q[c + i];
            std::string ga = q();
            L("or.b64 ", ga, ", ", gl, ", ", u64s(dm), ";");
            L("shl.b64 ", ga, ", ", ga, ", 3;");
            L("add.s64 ", ga, ", ", ga, ", %psi;");
            L("cp.async.bulk.global.shared::cta.bulk_group [", ga, "], [", sl, "+", (size_t)(m * 32 * rs), "], ", rs,
              ";");
        }
        L("cp.async.bulk.commit_group;");
        o << ls << ":\n";
    }
    uint32_t tlin_mask = 0;
    bool gen_pf = false;  // generic L2 prefetch (thread t -> 256 B chunk t of the next tile)

    // tile load (mapping m) from the tile at byte pointer `ptr` into registers <bank>0..R-1
    void reg_load(int m, const std::string& ptr, const std::string& bank) {
        std::string g = gb_of(m), ad = q();
        L("shl.b64 ", ad, ", ", g, ", ", ESL, ";");
        L("add.s64 ", ad, ", ", ad, ", ", ptr, ";");
        Bases B;
        for (int i = 0; i < R; ++i) {
            uint64_t off = 0;
            for (int b = 0; b < RB; ++b)
                if (i & (1 << b)) off |= 1ull << P.stg[m].reg_q[b];
            L("ld.global.cs.", CB, " ", bank, i, ", ", addr64(B, ad, off * ES), ";");
        }
    }

    // async tile load: global (mapping m, tile base register) -> SMEM buffer in
    // mapping m's layout (the layout a transpose out of m would write)
    void async_load(int m, const std::string& base) {
        const StageDesc& S = P.stg[m];
        std::string g = gb_of(m), ad = q(), pa = q();
        L("shl.b64 ", pa, ", ", base, ", 3;");
        L("add.s64 ", pa, ", ", pa, ", %psi;");
        L("shl.b64 ", ad, ", ", g, ", 3;");
        L("add.s64 ", ad, ", ", ad, ", ", pa, ";");
        std::string T = so_of(m);
        const uint32_t lm = thread_smask(m);
        Bases B;
        std::map<uint32_t, std::string> sb;
        for (int i = 0; i < R; ++i) {
            uint64_t off = 0;
            uint32_t so = 0;
            for (int b = 0; b < RB; ++b)
                if (i & (1 << b)) {
                    off |= 1ull << S.reg_q[b];
                    so ^= S.reg_s[b];
                }
            const uint32_t lo = so & lm, hi = so & ~lm;
            auto it = sb.find(lo);
            if (it == sb.end()) {
                std::string br = r();
                L("xor.b32 ", br, ", ", T, ", ", lo, ";");
                L("add.u32 ", br, ", ", br, ", %smb;");
                it = sb.emplace(lo, br).first;
            }
            L("cp.async.ca.shared.global [", it->second, "+", hi, "], ", addr64(B, ad, off * 8), ", 8;");
        }
        L("cp.async.commit_group;");
    }
    // called after each SMEM buffer read of a tile: after the last one, every
    // thread is done with the buffer and the next tile's loads may land in it
    void after_read() {
        if (pc) {
            if (--reads_left == 0) {
                std::string e = r();
                L("mad.lo.u32 ", e, ", %ib, 8, ", (unsigned)(tab_mb + 8 * kPcBufs), ";");
                L("add.u32 ", e, ", ", e, ", %smb;");
                L("mbarrier.arrive.shared::cta.b64 _, [", e, "];");
            }
            return;
        }
        if (!(variant & 1) || --reads_left != 0) return;
        std::string ls = lab();
        L("bar.sync 0;");
        L("@%pnext bra.uni ", ls, "_go;");
        L("bra.uni ", ls, ";");
        o << ls << "_go:\n";
        async_load(load_map, "%nbase");
        o << ls << ":\n";
    }
    int load_map = 0;
    int stagger_ns = 4000;
    uint64_t cmask_ = 0;

    // global stores of the tile through mapping si (register CX map and flips folded in)
    void store_stg(int si) {
        const StageDesc& S = P.stg[si];
        // slot bit b's global index vector: the stage's output mapping (its register CX
        // relabels), or its input mapping when the registers were transposed into it
        auto vec = [&](int b) { return st_in_ ? (1ull << S.reg_q[b]) : S.out_g[b]; };
        std::string g = gb_of(si);
        uint64_t lm = thread_gmask(si);
        std::string idx = g;
        if (fposs) {
            idx = q();
            L("mov.b64 ", idx, ", ", g, ";");
            for (int b = 0; b < RB; ++b) {
                if (!(fposs & (1u << b))) continue;
                std::string t = r(), t64 = q();
                L("bfe.u32 ", t, ", %F, ", b, ", 1;");
                L("cvt.u64.u32 ", t64, ", ", t, ";");
                L("neg.s64 ", t64, ", ", t64, ";");
                L("and.b64 ", t64, ", ", t64, ", ", u64s(vec(b)), ";");
                L("xor.b64 ", idx, ", ", idx, ", ", t64, ";");
                lm |= vec(b);
            }
        }
        std::map<uint64_t, std::pair<std::string, Bases>> bases;
        std::vector<std::pair<uint64_t, int>> order;  // variant 2097152: stores in ascending address
        for (int i = 0; i < R; ++i) {
            uint64_t og = 0;
            for (int b = 0; b < RB; ++b)
                if (i & (1 << b)) og ^= vec(b);
            order.push_back({og, i});
        }
        if (variant & 2097152) std::sort(order.begin(), order.end());
        for (const auto& oi : order) {
            const int i = oi.second;
            if (!in_sub(i)) continue;
            const uint64_t og = oi.first;
            const uint64_t lo = og & lm, hi = og & ~lm;
            auto it = bases.find(lo);
            if (it == bases.end()) {
                std::string x = q();
                if (lo) L("xor.b64 ", x, ", ", idx, ", ", u64s(lo), ";");
                else L("mov.b64 ", x, ", ", idx, ";");
                L("shl.b64 ", x, ", ", x, ", ", ESL, ";");
                if (variant & 1048576) {  // timing probe: stores into a 16 MiB L2-resident window
                    std::string y = q();
                    L("add.s64 ", y, ", ", x, ", %pt;");
                    L("sub.s64 ", y, ", ", y, ", %psi;");
                    L("and.b64 ", y, ", ", y, ", 0xffffff;");
                    L("add.s64 ", x, ", ", y, ", %psi;");
                } else {
                    L("add.s64 ", x, ", ", x, ", %pt;");
                }
                it = bases.emplace(lo, std::make_pair(x, Bases{})).first;
            }
            L((variant & 134217728) ? "st.global.wt." : (variant & 65536) ? "st.global." : "st.global.cs.", MT, " ",
              addr64(it->second.second, it->second.first, hi * ES), ", ", amem(a(i)), ";");
            if (il_) next_load(amap[i]);
        }
    }
    bool stored = false;
    bool st_in_ = false;  // store_stg: registers are in the stage's input mapping

    // store/load interleave: the register just stored receives the next tile's amplitude of
    // the load mapping's slot with the same register index, so the loads of tile t+1 stream
    // while tile t's stores drain (HBM keeps reads and writes in flight together)
    bool il_ = false;
    bool uph_il_ = false;  // interleave chosen for a pass with tile-uniform phase slots
    std::string nld_;   // byte address of the next tile in the load mapping (this thread)
    Bases nB_;
    void next_load(int phys) {
        if (nld_.empty()) {
            std::string g = gb_of(load_map), t = q();
            nld_ = q();
            L("shl.b64 ", t, ", %nbase, ", ESL, ";");
            L("add.s64 ", t, ", ", t, ", %psi;");
            L("shl.b64 ", nld_, ", ", g, ", ", ESL, ";");
            L("add.s64 ", nld_, ", ", nld_, ", ", t, ";");
            nB_ = Bases{};
        }
        uint64_t off = 0;
        for (int b = 0; b < RB; ++b)
            if (phys & (1 << b)) off |= 1ull << P.stg[load_map].reg_q[b];
        const std::string reg = (D ? "%A" : "%a") + std::to_string(phys);
        L((variant & 131072) ? "@%pnext ld.global." : "@%pnext ld.global.cs.", MT, " ", amem(reg), ", ",
          addr64(nB_, nld_, off * ES), ";");
    }

    // a run of consecutive phase ops (slot vectors W_k, factors e_k, no flip-vector
    // mixing) as ONE multiply per slot: slot p gets the product of the e_k with
    // parity(W_k & p) = 1; the per-class products are formed once per tile
    // (variant 16777216; same result up to the order of the complex products)
    void flush_ph_run(std::vector<std::pair<uint32_t, std::string>>& run) {
        if (run.empty()) return;
        if (run.size() == 1) {
            op_ph(run[0].first, run[0].second);
            run.clear();
            return;
        }
        const int m = (int)run.size();
        std::map<uint32_t, std::string> f;  // class -> product (packed)
        std::function<std::string(uint32_t)> prod = [&](uint32_t c) -> std::string {
            auto it = f.find(c);
            if (it != f.end()) return it->second;
            const int k0 = __builtin_ctz(c);
            std::string v;
            if ((c & (c - 1)) == 0) {
                v = run[k0].second;
            } else {
                const std::string rest = prod(c & (c - 1));
                auto [er2, ei2] = split_bc(run[k0].second);
                v = cv();
                c_mul(v, rest, er2, ei2);
            }
            f[c] = v;
            return v;
        };
        std::map<uint32_t, std::pair<std::string, std::string>> fb;  // class -> broadcast pair
        for (int i = 0; i < R; ++i) {
            if (!in_sub(i)) continue;
            uint32_t c = 0;
            for (int k2 = 0; k2 < m; ++k2) c |= (uint32_t)par(run[k2].first & (uint32_t)i) << k2;
            if (!c) continue;
            auto it = fb.find(c);
            if (it == fb.end()) it = fb.emplace(c, split_bc(prod(c))).first;
            c_mul(a(i), a(i), it->second.first, it->second.second);
        }
        run.clear();
    }

    // the op list and thread phases of stage s (slot filter applies)
    template <class TBF>
    bool stage_body(int s, TBF& TB) {
        const StageDesc& S = P.stg[s];
        std::vector<std::pair<uint32_t, std::string>> run;  // pending phase ops (variant 16777216)
        cur_stage = s;
        for (int oi = S.op_begin;; ++oi) {
            cur_op = oi;
            const uint32_t w = P.ops[oi];
            const uint32_t code = w & 0xffu;
            if (code >= dec.size() || dec[code].fam < 0) return false;
            if ((variant & 8) && dec[code].fam != 9) continue;  // timing probe: no ops (wrong results)
            const Dec d = dec[code];
            const uint32_t T = d.t >= 0 ? 1u << d.t : 0u, Cb = d.c >= 0 ? 1u << d.c : 0u;
            if (variant & 16777216) {
                if ((d.fam == F_PH || d.fam == F_PHW) && run.size() < 5) {
                    const uint32_t W = d.fam == F_PH ? T : (T | Cb);
                    if (!(W & fposs)) {
                        run.emplace_back(W, ph_product(w, TB()));
                        continue;
                    }
                }
                flush_ph_run(run);
            }
            if (d.fam == 9) break;
            switch (d.fam) {
                case F_RD: op_rd(T, T, w >> 16); break;
                case F_CD: op_cd(T, T, w >> 16); break;
                case F_PH: op_ph(T, ph_product(w, TB())); break;
                case F_RDW: op_rd(T, T | Cb, w >> 16); break;
                case F_RDV: op_rd(T | Cb, T, w >> 16); break;
                case F_PHW: op_ph(T | Cb, ph_product(w, TB())); break;
                case F_PH2: op_ph2(d.t, d.c, w >> 16); break;
                case 7: op_cxm(d.t, d.c); break;
                case 8: op_xf(w, TB()); break;
                default: return false;
            }
        }
        if (S.tph_end == S.tph_begin + 1 && !(variant & 8) && P.tph[S.tph_begin].cmask == 0 &&
            P.tph[S.tph_begin].qmask == 0 && P.tph[S.tph_begin].v[1] == 0 && P.tph[S.tph_begin].v[3] == 0 &&
            P.tph[S.tph_begin].v[0] == P.tph[S.tph_begin].v[2]) {
            // one unconditional real factor (a pass's rotation scale): a real multiply per
            // slot, the same values as the complex multiply by (v, 0) of the general path
            const std::string v = ldp_f32(tphv(S.tph_begin, 0));
            for (int i = 0; i < R; ++i) {
                if (!in_sub(i)) continue;
                if (!D) {
                    L("mul.rn.f32x2 ", a(i), ", ", a(i), ", ", bc(v), ";");
                } else {
                    auto [xr, xi] = unpack(a(i));
                    std::string nr = dq(), ni = dq();
                    L("mul.rn.f64 ", nr, ", ", xr, ", ", v, ";");
                    L("mul.rn.f64 ", ni, ", ", xi, ", ", v, ";");
                    pack_into(a(i), nr, ni);
                }
            }
        } else if (S.tph_end > S.tph_begin && !(variant & 8)) {
            std::string one = sv(), zero = sv();
            L("mov.", ST, " ", one, ", ", ONE, ";");
            L("mov.", ST, " ", zero, ", ", ZERO, ";");
            std::string ph = pack(one, zero);
            const std::string& t = TB();
            for (int e = S.tph_begin; e < S.tph_end; ++e) {
                const Entry<Real>& E = P.tph[e];
                std::string pc = p(), ph_ = p(), m1 = q(), m2 = q();
                L("and.b64 ", m1, ", ", t, ", ", u64s(E.cmask), ";");
                L("setp.eq.u64 ", pc, ", ", m1, ", ", u64s(E.cmask), ";");
                L("and.b64 ", m2, ", ", t, ", ", u64s(E.qmask), ";");
                L("setp.ne.u64 ", ph_, ", ", m2, ", 0;");
                std::string v0 = ldp_f32(tphv(e, 0)), v1 = ldp_f32(tphv(e, 1)), v2 = ldp_f32(tphv(e, 2)),
                            v3 = ldp_f32(tphv(e, 3));
                std::string vx = sv(), vy = sv(), np_ = cv();
                L("selp.", ST, " ", vx, ", ", v2, ", ", v0, ", ", ph_, ";");
                L("selp.", ST, " ", vy, ", ", v3, ", ", v1, ", ", ph_, ";");
                c_mul(np_, ph, bc(vx), bc(vy));
                ph = csel(np_, ph, pc);
            }
            auto [r2, i2] = split_bc(ph);
            for (int i = 0; i < R; ++i)
                if (in_sub(i)) c_mul(a(i), a(i), r2, i2);
        }
        return true;
    }

    // ---------------------------------------------------------------- prologue pieces
    // deposit the low bits of u32 x into the positions comp_q[0..n) (u64 result)
    std::string deposit(const std::string& x, int n) {
        std::string g = q();
        L("mov.u64 ", g, ", 0;");
        int i = 0;
        while (i < n) {
            int len = 1;
            while (i + len < n && P.comp_q[i + len] == P.comp_q[i] + len) ++len;
            std::string t = r(), t64 = q();
            L("bfe.u32 ", t, ", ", x, ", ", i, ", ", len, ";");
            L("cvt.u64.u32 ", t64, ", ", t, ";");
            L("shl.b64 ", t64, ", ", t64, ", ", (int)P.comp_q[i], ";");
            L("or.b64 ", g, ", ", g, ", ", t64, ";");
            i += len;
        }
        return g;
    }
    // per-thread global bits / SMEM offset of mapping m (prologue)
    void thread_map(int m, const std::string& lane, const std::string& warp, std::string& gb, std::string& so,
                    bool lanes = true, bool warps = true) {
        const StageDesc& S = P.stg[m];
        gb = q();
        so = r();
        L("mov.u64 ", gb, ", 0;");
        L("mov.u32 ", so, ", 0;");
        auto add = [&](const std::string& src, int bitn, int pos, uint32_t soff) {
            std::string t = r(), t64 = q(), m2 = r();
            L("bfe.u32 ", t, ", ", src, ", ", bitn, ", 1;");
            L("cvt.u64.u32 ", t64, ", ", t, ";");
            L("shl.b64 ", t64, ", ", t64, ", ", pos, ";");
            L("or.b64 ", gb, ", ", gb, ", ", t64, ";");
            L("neg.s32 ", m2, ", ", t, ";");
            L("and.b32 ", m2, ", ", m2, ", ", soff, ";");
            L("xor.b32 ", so, ", ", so, ", ", m2, ";");
        };
        if (lanes)
            for (int l = 0; l < kLaneBits; ++l) add(lane, l, S.lane_q[l], (uint32_t)S.lane_s[l] << ESL);
        if (warps)
            for (int w = 0; w < WB; ++w) add(warp, w, S.warp_q[w], (uint32_t)S.warp_s[w] << ESL);
    }

    std::string tb_of(int s) {  // base | rank_bits | thread bits of stage s
        std::string g = gb_of(s), t = q();
        L("or.b64 ", t, ", %base, %rk;");
        L("or.b64 ", t, ", ", t, ", ", g, ";");
        return t;
    }

    bool supported() const {
        if (NBUF != 1 || RB < 3 || RB > 6) return false;
        if (P.n_stages < 1 || P.n_stages > kMaxStages) return false;
        return true;
    }

    // the producer warp: fills buffer i % 3 with the CTA's tile i (mapping li's global
    // addresses, the common swizzled SMEM layout) once the consumers released its previous
    // contents; each lane's cp.async completions arrive on the buffer's full barrier
    void producer(int li, const std::string& lane, int n_comp) {
        o << "$PROD:\n";
        const StageDesc& S = P.stg[li];
        std::vector<std::string> gbv(1 << WB), sov(1 << WB);
        for (int w = 0; w < (1 << WB); ++w) {
            std::string wr = r();
            L("mov.u32 ", wr, ", ", w, ";");
            thread_map(li, lane, wr, gbv[w], sov[w], true, true);
            std::string gs = q();
            L("shl.b64 ", gs, ", ", gbv[w], ", ", ESL, ";");
            gbv[w] = gs;
        }
        L("ld.param.u64 %psi, [psi];");
        L("mov.u32 %pi, 0;");
        o << "$PLOOP:\n";
        std::string t = r(), t64 = q(), pp = p();
        L("mad.lo.u32 ", t, ", %pi, %nctile, %ctile;");
        L("cvt.u64.u32 ", t64, ", ", t, ";");
        L("setp.ge.u64 ", pp, ", ", t64, ", ", u64s(P.n_tiles), ";");
        L("@", pp, " bra.uni $PEND;");
        L("rem.u32 %pb, %pi, ", kPcBufs, ";");
        L("div.u32 %pj, %pi, ", kPcBufs, ";");
        {  // buffer reuse: its previous tile's group is done reading it
            std::string ls = lab(), lw = lab(), eb = r(), ph = r(), pz = p(), pw = p();
            L("setp.eq.u32 ", pz, ", %pj, 0;");
            L("@", pz, " bra.uni ", ls, ";");
            L("add.u32 ", ph, ", %pj, 1;");  // (j - 1) & 1
            L("and.b32 ", ph, ", ", ph, ", 1;");
            L("mad.lo.u32 ", eb, ", %pb, 8, ", (unsigned)(tab_mb + 8 * kPcBufs), ";");
            L("add.u32 ", eb, ", ", eb, ", %smb;");
            o << lw << ":\n";
            L("mbarrier.try_wait.parity.shared::cta.b64 ", pw, ", [", eb, "], ", ph, ";");
            L("@!", pw, " bra.uni ", lw, ";");
            o << ls << ":\n";
        }
        std::string base = deposit(t, n_comp), pt = q(), sbuf = r();
        L("shl.b64 ", pt, ", ", base, ", ", ESL, ";");
        L("add.s64 ", pt, ", ", pt, ", %psi;");
        L("mad.lo.u32 ", sbuf, ", %pb, ", (unsigned)buf_bytes, ", %smb;");
        const uint32_t lm = thread_smask(li);
        for (int w = 0; w < (1 << WB); ++w) {
            std::string ad = q();
            L("add.s64 ", ad, ", ", pt, ", ", gbv[w], ";");
            Bases B;
            std::map<uint32_t, std::string> sb;
            for (int i = 0; i < R; ++i) {
                uint64_t off = 0;
                uint32_t so = 0;
                for (int b = 0; b < RB; ++b)
                    if (i & (1 << b)) {
                        off |= 1ull << S.reg_q[b];
                        so ^= S.reg_s[b];
                    }
                const uint32_t lo = so & lm, hi = so & ~lm;
                auto it = sb.find(lo);
                if (it == sb.end()) {
                    std::string br = r();
                    L("xor.b32 ", br, ", ", sov[w], ", ", lo, ";");
                    L("add.u32 ", br, ", ", br, ", ", sbuf, ";");
                    it = sb.emplace(lo, br).first;
                }
                L("cp.async.ca.shared.global [", it->second, "+", hi, "], ", addr64(B, ad, off * ES), ", ", ES, ";");
            }
        }
        {
            std::string fb = r();
            L("mad.lo.u32 ", fb, ", %pb, 8, ", (unsigned)tab_mb, ";");
            L("add.u32 ", fb, ", ", fb, ", %smb;");
            L("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [", fb, "];");
        }
        L("add.u32 %pi, %pi, 1;");
        L("bra.uni $PLOOP;");
        o << "$PEND:\n";
        L("cp.async.wait_all;");
        L("ret;");
    }

    std::string run(const std::string& name) {
        const int ns = P.n_stages;
        const int li = P.load_direct ? 1 : 0;
        // variant 1073741824: stores go through the load mapping (one more transpose when the
        // last stage's mapping differs; in-place reads and writes of a tile then share one
        // HBM access order)
        const int si = (variant & 1073741824) ? li : P.store_direct ? ns : 0;
        const int n_comp = 63 - __builtin_clzll(P.n_tiles);
        uint64_t cmask = 0;
        for (int i = 0; i < n_comp; ++i) cmask |= 1ull << P.comp_q[i];
        cmask_ = cmask;
        if (std::getenv("QG_DEV_PLAN_DUMP")) {  // dev probe: io lanes of the load / store mappings
            std::fprintf(stderr, "uph %d ", P.n_uph);
            std::fprintf(stderr, "io ld %d st %d ns %d lanes_ld", P.load_direct, P.store_direct, ns);
            for (int l = 0; l < kLaneBits; ++l) std::fprintf(stderr, " %d", (int)P.stg[li].lane_q[l]);
            std::fprintf(stderr, " lanes_st");
            for (int l = 0; l < kLaneBits; ++l) std::fprintf(stderr, " %d", (int)P.stg[si].lane_q[l]);
            std::fprintf(stderr, "\n");
        }

        // ---- prologue
        if (pc) {  // consumers: thread index within the group (both groups share the per-thread tables)
            L("mov.u32 %xtidf, %tid.x;");
            L("and.b32 %xtid, %xtidf, ", NT - 1, ";");
        } else {
            L("mov.u32 %xtid, %tid.x;");
        }
        std::string lane = r(), warp = r();
        L("and.b32 ", lane, ", %xtid, 31;");
        L("shr.u32 ", warp, ", %xtid, 5;");
        L("mov.u32 %xlane, ", lane, ";");
        L("mov.u32 %xwarp, ", warp, ";");
        // scoped hand-over barriers (see hand_sync): off for the probe / alternative forms
        // that share the buffer differently, and for tile-uniform phase slots (their
        // per-tile table is written by one warp and read by all)
        {
            static const bool off = std::getenv("QG_DEV_CTA_SYNC") != nullptr;  // A/B probe
            wsync_ = !off && !pc && NBUF == 1 && WB == 3 && P.n_uph == 0 &&
                     !(variant & (1 | 4096 | 8192 | 262144 | 16 | 32 | 16384 | 67108864));
            if (wsync_) {
                int cur = li;
                for (int s2 = 1; s2 <= ns; ++s2)
                    if (cur != s2) { last_dst_ = s2; cur = s2; }
                if (cur != si) last_dst_ = si;
                for (int j = 0; j < 3; ++j) {  // 1 + 4j + (warp index without bit j)
                    std::string lo = r(), hi = r();
                    L("and.b32 ", lo, ", ", warp, ", ", (1 << j) - 1, ";");
                    L("shr.u32 ", hi, ", ", warp, ", ", j + 1, ";");
                    L("shl.b32 ", hi, ", ", hi, ", ", j, ";");
                    L("or.b32 ", lo, ", ", lo, ", ", hi, ";");
                    L("add.u32 %gid", j, ", ", lo, ", ", 1 + 4 * j, ";");
                }
            }
        }
        L("mov.u32 %smb, smem;");
        L("add.u32 %smb2, %smb, ", buf_bytes, ";");
        // per-mapping tables of the lane and warp parts of a thread's global bits and
        // SMEM offset (a thread's value = lane part | warp part); warp 0 writes the lane
        // entries, lane 0 of every warp its warp's entries
        auto base_reg = [&](const char* reg, const std::string& idx, int scale) {
            L("shl.b32 ", reg, ", ", idx, ", ", scale, ";");
            L("add.u32 ", reg, ", ", reg, ", %smb;");
            L("add.u32 ", reg, ", ", reg, ", ", tab_gb, ";");
        };
        base_reg("%tl8", lane, 3);
        base_reg("%tw8", warp, 3);
        base_reg("%tl4", lane, 2);
        base_reg("%tw4", warp, 2);
        L("setp.eq.u32 %pw0, ", warp, ", 0;");
        L("setp.eq.u32 %pl0, ", lane, ", 0;");
        if (variant & 524288)
            for (int m = 0; m <= ns; ++m) {
                std::string g, so;
                thread_map(m, lane, warp, g, so, true, true);
                L("mov.b64 %gbm", m, ", ", g, ";");
                L("mov.b32 %som", m, ", ", so, ";");
            }
        for (int m = 0; m <= ns; ++m) {
            std::string gl, sl, gw, sw;
            thread_map(m, lane, warp, gl, sl, true, false);
            thread_map(m, lane, warp, gw, sw, false, true);
            L("@%pw0 st.shared.u64 [%tl8+", (size_t)m * kMapBytes, "], ", gl, ";");
            L("@%pw0 st.shared.u32 [%tl4+", (size_t)m * kMapBytes + 384, "], ", sl, ";");
            L("@%pl0 st.shared.u64 [%tw8+", (size_t)m * kMapBytes + 256, "], ", gw, ";");
            L("@%pl0 st.shared.u32 [%tw4+", (size_t)m * kMapBytes + 512, "], ", sw, ";");
        }
        {  // L2 prefetch offset: lanes < R cover the register runs of the io load mapping
            const StageDesc& S = P.stg[li];
            std::string g = q(), gw = q();
            L("mov.u64 ", gw, ", 0;");
            for (int w = 0; w < WB; ++w) {
                std::string t = r(), t64 = q();
                L("bfe.u32 ", t, ", ", warp, ", ", w, ", 1;");
                L("cvt.u64.u32 ", t64, ", ", t, ";");
                L("shl.b64 ", t64, ", ", t64, ", ", (int)S.warp_q[w], ";");
                L("or.b64 ", gw, ", ", gw, ", ", t64, ";");
            }
            L("mov.u64 ", g, ", 0;");
            for (int b = 0; b < RB; ++b) {
                std::string t = r(), t64 = q();
                L("bfe.u32 ", t, ", ", lane, ", ", b, ", 1;");
                L("cvt.u64.u32 ", t64, ", ", t, ";");
                L("shl.b64 ", t64, ", ", t64, ", ", (int)S.reg_q[b], ";");
                L("or.b64 ", g, ", ", g, ", ", t64, ";");
            }
            const size_t pf = tab_pf - tab_gb;
            L("@%pw0 st.shared.u64 [%tl8+", pf, "], ", g, ";");
            L("@%pl0 st.shared.u64 [%tw8+", pf + 256, "], ", gw, ";");
        }
        L("setp.lt.u32 %pfl, ", lane, ", ", R, ";");
        if (!hoist_ops.empty()) {  // per-thread products of the thread-constant phase factors
            L("shl.b32 %hpb, %xtid, ", ESL, ";");
            L("add.u32 %hpb, %hpb, %smb;");
            L("add.u32 %hpb, %hpb, ", tab_hp, ";");
            std::string rk = q();
            L("ld.param.u64 ", rk, ", [rk];");
            prologue_ = true;
            for (size_t h = 0; h < hoist_ops.size(); ++h) {
                const int s2 = hoist_ops[h].first, oi = hoist_ops[h].second;
                std::string g, so, tb = q();
                thread_map(s2, lane, warp, g, so, true, true);
                L("or.b64 ", tb, ", ", g, ", ", rk, ";");
                std::string e = hoisted_product(s2, P.ops[oi], tb);
                L("st.shared.", CB, " [%hpb+", h * (size_t)NT * ES, "], ", e, ";");
            }
            prologue_ = false;
        }
        gen_pf = run_bits() >= 5 && (1 << (k - 5)) == NT;
        if (gen_pf) {  // thread t prefetches 256 B chunk t of the next tile (whatever the mappings)
            L("mov.u64 %pfg, 0;");
            for (int i = 0; i < k - 5; ++i) {
                std::string t = r(), t64 = q();
                L("bfe.u32 ", t, ", %xtid, ", i, ", 1;");
                L("cvt.u64.u32 ", t64, ", ", t, ";");
                L("shl.b64 ", t64, ", ", t64, ", ", (int)P.tile_q[5 + i], ";");
                L("or.b64 %pfg, %pfg, ", t64, ";");
            }
            L("setp.eq.u32 %pfl, 1, 1;");
        }
        if (variant & 262144) {
            const StageDesc& S = P.stg[si];
            L("mov.u32 %tlin, 0;");
            auto addl = [&](const std::string& src, int bitn, uint32_t off) {
                std::string t = r();
                L("bfe.u32 ", t, ", ", src, ", ", bitn, ", 1;");
                L("neg.s32 ", t, ", ", t, ";");
                L("and.b32 ", t, ", ", t, ", ", off, ";");
                L("xor.b32 %tlin, %tlin, ", t, ";");
                tlin_mask |= off;
            };
            for (int l = 0; l < kLaneBits; ++l) addl(lane, l, swz(S.lane_s[l]) << 3);
            for (int w = 0; w < WB; ++w) addl(warp, w, swz(S.warp_s[w]) << 3);
            const int c = run_bits(), nrb = k - c;
            L("mov.u64 %rdl, 0;");
            for (int i = 0; i < nrb && i < 5; ++i) {
                std::string t = r(), t64 = q();
                L("bfe.u32 ", t, ", ", lane, ", ", i, ", 1;");
                L("cvt.u64.u32 ", t64, ", ", t, ";");
                L("shl.b64 ", t64, ", ", t64, ", ", (int)P.tile_q[c + i], ";");
                L("or.b64 %rdl, %rdl, ", t64, ";");
            }
        }
        if (pc) {
            std::string ls = lab(), pp = p();
            L("setp.ne.u32 ", pp, ", %xtidf, 0;");
            L("@", pp, " bra.uni ", ls, ";");
            for (int b = 0; b < kPcBufs; ++b) {
                L("mbarrier.init.shared::cta.b64 [smem+", tab_mb + 8 * b, "], 32;");             // full: producer lanes
                L("mbarrier.init.shared::cta.b64 [smem+", tab_mb + 8 * (kPcBufs + b), "], ", NT, ";");  // empty
            }
            o << ls << ":\n";
        }
        L("bar.sync 0;");
        L("mov.u32 %ctile, %ctaid.x;");
        L("mov.u32 %nctile, %nctaid.x;");
        if (pc) {
            L("setp.ge.u32 %ppr, %xtidf, ", 2 * NT, ";");
            L("@%ppr bra.uni $PROD;");
            std::string g = r(), t0 = r(), g2 = r();
            L("shr.u32 ", g, ", %xtidf, ", 5 + WB, ";");
            L("add.u32 %gbar, ", g, ", 1;");
            L("mad.lo.u32 ", t0, ", ", g, ", %nctile, %ctile;");
            L("shl.b32 ", g2, ", %nctile, 1;");
            L("cvt.u64.u32 %tile, ", t0, ";");
            L("cvt.u64.u32 %G, ", g2, ";");
            L("mov.u64 %tend, ", u64s(P.n_tiles), ";");
            std::string b0 = deposit(t0, n_comp), dg = deposit(g2, n_comp);
            L("mov.u64 %base, ", b0, ";");
            L("mov.u64 %dG, ", dg, ";");
            L("mov.u32 %ii, ", g, ";");
        } else if (variant & 4) {  // contiguous tile ranges per CTA: consecutive tiles are adjacent runs
            std::string c64 = q(), g64 = q(), t0 = q(), t1 = q(), t0s = r();
            L("cvt.u64.u32 ", c64, ", %ctile;");
            L("cvt.u64.u32 ", g64, ", %nctile;");
            L("mul.lo.u64 ", t0, ", ", c64, ", ", u64s(P.n_tiles), ";");
            L("div.u64 ", t0, ", ", t0, ", ", g64, ";");
            L("add.s64 ", t1, ", ", c64, ", 1;");
            L("mul.lo.u64 ", t1, ", ", t1, ", ", u64s(P.n_tiles), ";");
            L("div.u64 %tend, ", t1, ", ", g64, ";");
            L("mov.u64 %tile, ", t0, ";");
            L("mov.u64 %G, 1;");
            L("cvt.u32.u64 ", t0s, ", ", t0, ";");
            std::string b0 = deposit(t0s, n_comp);
            L("mov.u64 %base, ", b0, ";");
            L("mov.u64 %dG, ", u64s(n_comp > 0 ? (1ull << P.comp_q[0]) : 0), ";");
        } else {
            L("cvt.u64.u32 %tile, %ctile;");
            L("cvt.u64.u32 %G, %nctile;");
            L("mov.u64 %tend, ", u64s(P.n_tiles), ";");
            std::string b0 = deposit("%ctile", n_comp), dg = deposit("%nctile", n_comp);
            L("mov.u64 %base, ", b0, ";");
            L("mov.u64 %dG, ", dg, ";");
        }
        L("ld.param.u64 %psi, [psi];");
        L("ld.param.u64 %rk, [rk];");
        if (variant & 64) {  // desynchronise the CTAs sharing an SM: the second half starts late
            std::string h = r(), pp = p(), ls = lab();
            L("shr.u32 ", h, ", %nctile, 1;");
            L("setp.lt.u32 ", pp, ", %ctile, ", h, ";");
            L("@", pp, " bra.uni ", ls, ";");
            L("nanosleep.u32 ", stagger_ns, ";");
            o << ls << ":\n";
        }
        load_map = li;
        if (variant & 1) {  // the CTA's first tile
            std::string ls = lab();
            L("setp.ge.u64 %pend, %tile, %tend;");
            L("@%pend bra.uni ", ls, ";");
            async_load(li, "%base");
            o << ls << ":\n";
        }
        if (variant & 4096) {  // the CTA's first tile into the prefetch bank
            std::string ls = lab(), pt0 = q();
            L("setp.ge.u64 %pend, %tile, %tend;");
            L("@%pend bra.uni ", ls, ";");
            L("shl.b64 ", pt0, ", %base, ", ESL, ";");
            L("add.s64 ", pt0, ", ", pt0, ", %psi;");
            reg_load(li, pt0, "%b");
            o << ls << ":\n";
        }

        // passes with tile-uniform phase slots (QFT-like: a long per-tile prologue) stream better
        // with the store/load interleave and without the L2 prefetch (QFT28 2.95 -> 2.84 ms);
        // the random-circuit passes keep the prefetch (interleave + no prefetch: +1 %)
        static const bool no_uph_il = std::getenv("QG_DEV_NO_UPH_IL") != nullptr;  // A/B probe
        uph_il_ = P.n_uph > 0 && !no_uph_il;
        il_ = ((variant & 536870912) || uph_il_) && !(variant & (1 | 4096 | 32 | 32768 | 16384 | 262144 | 1048576));
        if (il_) {  // the CTA's first tile (later tiles are loaded by the previous tile's stores)
            std::string ls = lab(), pt0 = q();
            L("setp.ge.u64 %pend, %tile, %tend;");
            L("@%pend bra.uni ", ls, ";");
            L("shl.b64 ", pt0, ", %base, ", ESL, ";");
            L("add.s64 ", pt0, ", ", pt0, ", %psi;");
            for (int i = 0; i < R; ++i) amap[i] = i;
            std::string g = gb_of(li), ad = q();
            L("shl.b64 ", ad, ", ", g, ", ", ESL, ";");
            L("add.s64 ", ad, ", ", ad, ", ", pt0, ";");
            Bases B;
            for (int i = 0; i < R; ++i) {
                uint64_t off = 0;
                for (int b = 0; b < RB; ++b)
                    if (i & (1 << b)) off |= 1ull << P.stg[li].reg_q[b];
                L((variant & 131072) ? "ld.global." : "ld.global.cs.", MT, " ", amem(a(i)), ", ", addr64(B, ad, off * ES),
                  ";");
            }
            o << ls << ":\n";
        }

        // ---- tile loop
        o << "$LOOP:\n";
        L("setp.ge.u64 %pend, %tile, %tend;");
        L("@%pend bra.uni $END;");
        L("shl.b64 %pt, %base, ", ESL, ";");
        L("add.s64 %pt, %pt, %psi;");
        L("add.s64 %ntile, %tile, %G;");
        L("or.b64 %nbase, %base, ", u64s(~cmask), ";");
        L("add.s64 %nbase, %nbase, %dG;");
        L("and.b64 %nbase, %nbase, ", u64s(cmask), ";");
        L("setp.lt.u64 %pnext, %ntile, %tend;");
        first_tr = true;
        tbuf = 0;
        nld_.clear();
        if (pc) {
            // tile i of the CTA lives in buffer i % 3 (its (i / 3)-th fill): wait for the
            // producer, then read stage 1's mapping straight out of the buffer
            std::string j = r(), ph = r(), fb = r(), pp = p(), lw = lab();
            L("rem.u32 %ib, %ii, ", kPcBufs, ";");
            L("div.u32 ", j, ", %ii, ", kPcBufs, ";");
            L("and.b32 ", ph, ", ", j, ", 1;");
            L("mad.lo.u32 %smc, %ib, ", (unsigned)buf_bytes, ", %smb;");
            L("mad.lo.u32 ", fb, ", %ib, 8, ", (unsigned)tab_mb, ";");
            L("add.u32 ", fb, ", ", fb, ", %smb;");
            o << lw << ":\n";
            L("mbarrier.try_wait.parity.shared::cta.b64 ", pp, ", [", fb, "], ", ph, ";");
            L("@!", pp, " bra.uni ", lw, ";");
            reads_left = 1 + (ns - 1) + (P.store_direct ? 0 : 1);
            std::vector<uint32_t> O(R);
            for (int i = 0; i < R; ++i) {
                uint32_t v = 0;
                for (int b = 0; b < RB; ++b)
                    if (i & (1 << b)) v ^= P.stg[1].reg_s[b];
                O[i] = v;
            }
            smem_load(so_of(1), thread_smask(1), O, "%smc");
            after_read();
        } else if (il_) {
            // this tile's registers were loaded by the previous tile's stores (or before the loop)
        } else if (variant & 4096) {  // this tile from the prefetch bank; the next tile's loads into it
            for (int i = 0; i < R; ++i) L("mov.b64 ", a(i), ", %b", i, ";");
            std::string ls = lab(), pn = q();
            L("@!%pnext bra.uni ", ls, ";");
            L("shl.b64 ", pn, ", %nbase, ", ESL, ";");
            L("add.s64 ", pn, ", ", pn, ", %psi;");
            reg_load(li, pn, "%b");
            o << ls << ":\n";
        } else if (variant & 1) {  // this tile was loaded into the SMEM buffer by cp.async; read stage 1's mapping
            L("cp.async.wait_all;");
            L("bar.sync 0;");
            reads_left = 1 + (ns - 1) + (P.store_direct ? 0 : 1);
            std::vector<uint32_t> O(R);
            for (int i = 0; i < R; ++i) {
                uint32_t v = 0;
                for (int b = 0; b < RB; ++b)
                    if (i & (1 << b)) v ^= P.stg[1].reg_s[b];
                O[i] = v;
            }
            smem_load(so_of(1), thread_smask(1), O);
            after_read();
        } else if (variant & (32 | 32768)) {  // timing probes: no global loads (wrong results)
            for (int i = 0; i < R; ++i) {
                std::string z = sv();
                L("mov.", ST, " ", z, ", ", ZERO, ";");
                pack_into(a(i), z, z);
            }
        } else {  // load (io or stage-1 mapping): thread bits and register bits are disjoint
            std::string g = gb_of(li), ad = q();
            L("shl.b64 ", ad, ", ", g, ", ", ESL, ";");
            L("add.s64 ", ad, ", ", ad, ", %pt;");
            Bases B;
            for (int i = 0; i < R; ++i) {
                uint64_t off = 0;
                for (int b = 0; b < RB; ++b)
                    if (i & (1 << b)) off |= 1ull << P.stg[li].reg_q[b];
                L((variant & 131072) ? "ld.global." : "ld.global.cs.", MT, " ", amem(a(i)), ", ", addr64(B, ad, off * ES), ";");
            }
        }
        if (!(variant & 128) && !pc && !(uph_il_ && il_)) {  // warm L2 with this CTA's next tile (variant 512: the one after)
            std::string pp = p(), pf = q(), ad = q();
            std::string tgt = "%nbase";
            if (variant & (512 | 4096)) {
                std::string t2 = q(), nb2 = q();
                pp = p();
                L("add.s64 ", t2, ", %ntile, %G;");
                L("setp.lt.u64 ", pp, ", ", t2, ", %tend;");
                L("and.pred ", pp, ", ", pp, ", %pfl;");
                L("or.b64 ", nb2, ", %nbase, ", u64s(~cmask_), ";");
                L("add.s64 ", nb2, ", ", nb2, ", %dG;");
                L("and.b64 ", nb2, ", ", nb2, ", ", u64s(cmask_), ";");
                tgt = nb2;
            } else {
                L("and.pred ", pp, ", %pnext, %pfl;");
            }
            std::string ls = lab();
            L("@!", pp, " bra.uni ", ls, ";");
            if (gen_pf) {
                L("mov.b64 ", pf, ", %pfg;");
            } else {
                const size_t pfo = tab_pf - tab_gb;
                std::string a1 = q(), a2 = q();
                L("ld.shared.u64 ", a1, ", [%tl8+", pfo, "];");
                L("ld.shared.u64 ", a2, ", [%tw8+", pfo + 256, "];");
                L("or.b64 ", pf, ", ", a1, ", ", a2, ";");
            }
            L("or.b64 ", ad, ", ", pf, ", ", tgt, ";");
            L("shl.b64 ", ad, ", ", ad, ", ", ESL, ";");
            L("add.s64 ", ad, ", ", ad, ", %psi;");
            if (variant & 256) {
                L("cp.async.bulk.prefetch.L2.global [", ad, "], 256;");
            } else if (variant & 1024) {  // 64 B granules
                for (int o2 = 0; o2 < 256; o2 += 64) L("prefetch.global.L2 [", ad, "+", o2, "];");
            } else {  // one 32-amplitude chunk: 2 (complex64) / 4 (complex128) lines
                for (int o2 = 0; o2 < 32 * ES; o2 += 128)
                    L((variant & 268435456) ? "prefetch.global.L2::evict_last [" : "prefetch.global.L2 [", ad, "+", o2, "];");
            }
            o << ls << ":\n";
        }
        if (P.n_uph > 0) {  // tile-uniform phase slots: one warp per slot, lanes split the factors
            std::string ub = q(), pb = q();
            L("or.b64 ", ub, ", %base, %rk;");
            L("mov.b64 ", pb, ", P;");
            L("bar.sync 0;");  // every thread is done with the previous tile's slots
            for (int u = 0; u < P.n_uph; ++u) {
                const uint32_t d = P.uph[u];
                const int first = (int)(d & 0xffffu), cnt = (int)(d >> 16);
                std::string ls = lab(), pp = p();
                L("setp.ne.u32 ", pp, ", %xwarp, ", u % (NT / 32), ";");
                L("@", pp, " bra.uni ", ls, ";");
                std::string one = sv(), zero = sv();
                L("mov.", ST, " ", one, ", ", ONE, ";");
                L("mov.", ST, " ", zero, ", ", ZERO, ";");
                std::string e = pack(one, zero);
                for (int r0 = 0; r0 < cnt; r0 += 32) {
                    // entry first + r0 + lane (runtime index into the param space)
                    std::string idx = r(), off = q(), ad = q(), pos = r(), ex = sv(), ey = sv();
                    std::string inr = p(), on = p(), t = q(), tb = r();
                    L("setp.lt.u32 ", inr, ", %xlane, ", cnt - r0, ";");
                    L("add.u32 ", idx, ", %xlane, ", first + r0, ";");
                    L("mul.wide.u32 ", off, ", ", idx, ", ", sizeof(PhEnt<Real>), ";");
                    L("add.s64 ", ad, ", ", pb, ", ", off, ";");
                    L("add.s64 ", ad, ", ", ad, ", ", off_ph, ";");
                    L("@", inr, " ld.param.u32 ", pos, ", [", ad, "];");
                    L("@", inr, " ld.param.", ST, " ", ex, ", [", ad, "+", offsetof(PhEnt<Real>, e), "];");
                    L("@", inr, " ld.param.", ST, " ", ey, ", [", ad, "+", offsetof(PhEnt<Real>, e) + sizeof(Real), "];");
                    L("@!", inr, " mov.u32 ", pos, ", 0;");
                    L("shr.b64 ", t, ", ", ub, ", ", pos, ";");
                    L("cvt.u32.u64 ", tb, ", ", t, ";");
                    L("and.b32 ", tb, ", ", tb, ", 1;");
                    L("setp.ne.u32 ", on, ", ", tb, ", 0;");
                    L("and.pred ", on, ", ", on, ", ", inr, ";");
                    std::string ne = cv();
                    std::string vr = bc(ex), vi = bc(ey);
                    c_mul(ne, e, vr, vi);
                    e = csel(ne, e, on);
                }
                for (int o2 = 16; o2; o2 >>= 1) {  // product tree over the lanes
                    auto [ex, ey] = unpack(e);
                    std::string sx = shfl_s(ex, o2), sy = shfl_s(ey, o2), ne = cv();
                    c_mul(ne, e, bc(sx), bc(sy));
                    e = ne;
                }
                std::string ad = r();
                L("add.u32 ", ad, ", %smb, ", tab_uph + ES * (size_t)u, ";");
                L("@%pl0 st.shared.", CB, " [", ad, "], ", e, ";");
                o << ls << ":\n";
            }
            L("bar.sync 0;");
        }
        L("mov.u32 %F, 0;");
        fposs = 0;
        for (int i = 0; i < R; ++i) amap[i] = i;
        int cur = ((variant & 1) || pc) ? 1 : li;
        for (int s = 1; s <= ns; ++s) {
            const StageDesc& S = P.stg[s];
            if (cur != s && !(variant & 16)) {  // (variant 16: timing probe without transposes)
                transpose(cur, s);
                cur = s;
            }
            std::string tb;  // lazily
            auto TB = [&]() -> const std::string& {
                if (tb.empty()) tb = tb_of(s);
                return tb;
            };
            const bool split = (variant & 4194304) && s == ns && si == ns && !(variant & (8 | 16 | 32 | 16384 | 262144));
            uint32_t spect = 0;  // register bits no pair op / register move of this stage couples
            if (split) {
                uint32_t touched = 0;
                for (int oi = S.op_begin;; ++oi) {
                    const uint32_t code = P.ops[oi] & 0xffu;
                    if (code >= dec.size() || dec[code].fam < 0) return "";
                    const Dec d = dec[code];
                    if (d.fam == 9) break;
                    const uint32_t T = d.t >= 0 ? 1u << d.t : 0u, Cb = d.c >= 0 ? 1u << d.c : 0u;
                    if (d.fam == F_RD || d.fam == F_CD || d.fam == F_RDW) touched |= T;
                    if (d.fam == F_RDV) touched |= T | Cb;
                    if (d.fam == 7) touched |= T | Cb;
                }
                for (int b = RB - 1; b >= 0 && __builtin_popcount(spect) < 2; --b)
                    if (!(touched & (1u << b))) spect |= 1u << b;
            }
            if (!spect) {
                if (!stage_body(s, TB)) return "";
            } else {
                // the last stage in independent slot subsets (fixed spectator bits), each
                // stored as soon as it is final: the STG burst interleaves with the compute
                // of the next subset.  Register renames, the flip vector and its static
                // knowledge restart from the same state for every subset.
                std::string F0 = r();
                L("mov.u32 ", F0, ", %F;");
                int amap0[64];
                std::copy(amap, amap + R, amap0);
                const uint32_t fposs0 = fposs;
                const int nsub = 1 << __builtin_popcount(spect);
                for (int k2 = 0; k2 < nsub; ++k2) {
                    uint32_t v = 0;
                    for (int b = 0, t = 0; b < RB; ++b)
                        if (spect & (1u << b)) v |= (uint32_t)((k2 >> t++) & 1) << b;
                    fmask = spect;
                    fval = v;
                    if (k2) {
                        L("mov.u32 %F, ", F0, ";");
                        std::copy(amap0, amap0 + R, amap);
                        fposs = fposs0;
                    }
                    if (!stage_body(s, TB)) return "";
                    store_stg(si);
                }
                fmask = fval = 0;
                stored = true;
            }
        }
        if (cur != si && !(variant & 16)) {
            transpose(cur, si);
            cur = si;
            st_in_ = si != 0;
        }
        if ((variant & 262144) && !(variant & (32 | 16384))) {
            tma_store(si);
        } else if (!(variant & (32 | 16384)) && !stored) {
            store_stg(si);
        }
        stored = false;
        st_in_ = false;
        L("mov.u64 %tile, %ntile;");
        L("mov.u64 %base, %nbase;");
        if (pc) L("add.u32 %ii, %ii, 2;");
        L("bra.uni $LOOP;");
        o << "$END:\n";
        if (variant & 262144) L("cp.async.bulk.wait_group 0;");
        L("ret;");
        if (pc) producer(li, lane, n_comp);

        // ---- header
        std::ostringstream h;
        h << ".version 8.8\n.target sm_100a\n.address_size 64\n\n";
        h << ".extern .shared .align 16 .b8 smem[];\n\n";
        h << ".visible .entry " << name << "(\n\t.param .align 8 .b8 P[" << sizeof(PD)
          << "],\n\t.param .u64 psi,\n\t.param .u64 rk\n)\n";
        int min_ctas = (D || WB >= 4 || RB >= 6 || (variant & (2048 | 4096))) ? 1 : ((variant & 2) ? 3 : 2);
        if (variant & 8388608) min_ctas = 3;  // probe: three CTAs per SM (register cap 65536 / (3 x threads))
        if (pc) min_ctas = 1;
        if (!D && RB == 4 && WB == 4 && std::getenv("QG_DEV_JIT_CFG0")) min_ctas = 2;  // probe: 2 x 16 warps / SM
        if (!D && RB == 4 && WB == 3 && std::getenv("QG_DEV_JIT_CFG0")) min_ctas = 4;  // probe: 4 x 8 warps / SM
        if (D && RB == 4 && WB == 3 && std::getenv("QG_DEV_JIT_CFG0")) min_ctas = 2;   // probe: c128, 2 x 8 warps / SM
        h << ".maxntid " << (pc ? 2 * NT + 32 : NT) << ", 1, 1\n.minnctapersm " << min_ctas << "\n{\n";
        if (pc) h << "\t.reg .b32 %xtidf, %gbar, %smc, %ii, %ib, %pi, %pb, %pj, %pt32;\n\t.reg .pred %ppr;\n";
        if (D) h << "\t.reg .f64 %ar<" << R << ">, %ai<" << R << ">;\n";
        else h << "\t.reg .b64 %a<" << R << ">;\n";
        h << "\t.reg .b128 %x<" << (nx + 1) << ">;\n\t.reg .f64 %d<" << (nd + 1) << ">;\n";
        if (variant & 4096) h << "\t.reg .b64 %b<" << R << ">;\n";
        h << "\t.reg .b64 %q<" << (nq + 1) << ">;\n";
        h << "\t.reg .b32 %r<" << (nr + 1) << ">;\n";
        h << "\t.reg .f32 %f<" << (nf + 1) << ">;\n";
        h << "\t.reg .pred %p<" << (np + 1) << ">;\n";
        h << "\t.reg .b32 %xtid, %xlane, %xwarp, %smb, %smb2, %tlin, %tl8, %tw8, %tl4, %tw4, %F, %ctile, %nctile, %gid0, %gid1, %gid2;\n";
        h << "\t.reg .b64 %rdl, %pfg;\n\t.reg .b32 %hpb;\n";
        h << "\t.reg .b64 %gbm<" << (P.n_stages + 1) << ">;\n\t.reg .b32 %som<" << (P.n_stages + 1) << ">;\n";
        h << "\t.reg .b64 %tile, %tend, %ntile, %G, %base, %nbase, %dG, %psi, %rk, %pt;\n";
        h << "\t.reg .pred %pfl, %pend, %pnext, %pw0, %pl0;\n";
        return h.str() + o.str() + "}\n";
    }
};

}  // namespace

int jit_variant() {
    static const int v = [] {
        // default: per-thread mapping values in registers (524288) and the last stage in
        // slot subsets with interleaved stores (4194304) and thread-constant phase factors
        // hoisted to the prologue (33554432); the other bits are
        // measurement probes (tools/jit_time.py, profiles/r02*_jit_variants*.jsonl)
        const char* e = std::getenv("QG_JIT_VARIANT");
        return e ? std::atoi(e) : (524288 | 4194304 | 33554432);
    }();
    return v;
}

template <typename Real>
std::string jit_ptx(const PassDesc<Real>& P, int rb, int wb, int nbuf, const std::string& name) {
    Gen<Real> g(P, rb, wb, nbuf, jit_variant());
    if (const char* e = std::getenv("QG_JIT_STAGGER_NS")) g.stagger_ns = std::atoi(e);
    if (!g.supported()) return "";
    g.plan_hoist();
    if (g.pc_use()) g.enable_pc();
    return g.run(name);
}
template std::string jit_ptx<float>(const PassDesc<float>&, int, int, int, const std::string&);
template std::string jit_ptx<double>(const PassDesc<double>&, int, int, int, const std::string&);

template <typename Real>
size_t jit_smem_bytes(const PassDesc<Real>& P, int rb, int wb, int nbuf) {
    Gen<Real> g(P, rb, wb, nbuf, jit_variant());
    g.plan_hoist();
    if (g.pc_use()) return Gen<Real>::pc_smem_bytes(P) + g.hoist_bytes();
    return Gen<Real>::smem_bytes(P, rb, wb, nbuf, g.variant) + g.hoist_bytes();
}

template <typename Real>
int jit_block_threads(const PassDesc<Real>& P, int rb, int wb, int nbuf) {
    Gen<Real> g(P, rb, wb, nbuf, jit_variant());
    g.plan_hoist();
    return g.pc_use() ? 2 * (32 << wb) + 32 : (32 << wb);
}

// Process-wide cache of compiled passes keyed by their PTX text: re-planning the
// same circuit (run_circuit called again, batched rebinding with unchanged
// parameters, bench steps) reuses the cubins instead of recompiling.
namespace {
std::mutex g_cache_mu;
// never destroyed: modules would otherwise unload their libraries after the CUDA
// runtime has shut down at process exit
auto& g_cache = *new std::unordered_map<std::string, std::shared_ptr<JitModule>>();
size_t g_cache_bytes = 0;
constexpr size_t kCacheMaxBytes = (size_t)1 << 30;  // PTX + cubin bytes kept

// (a module stays loaded while any plan or the cache holds it; loaded libraries are
// reused by every later plan with the same pass: no per-plan cudaLibraryLoadData)
std::shared_ptr<JitModule> cache_get(const std::string& ptx) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(ptx);
    return it == g_cache.end() ? nullptr : it->second;
}
void cache_put(const std::string& ptx, const std::shared_ptr<JitModule>& m) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    if (g_cache_bytes + ptx.size() + m->cubin.size() > kCacheMaxBytes) {
        g_cache.clear();
        g_cache_bytes = 0;
    }
    if (g_cache.emplace(ptx, m).second) g_cache_bytes += ptx.size() + m->cubin.size();
}
}  // namespace

int64_t jit_cache_hits() { return g_cache_hits.load(); }

namespace {
struct DescHit {
    std::shared_ptr<JitModule> mod;
    size_t smem = 0;
    int threads = 0;
};
std::mutex g_dcache_mu;
auto& g_dcache = *new std::unordered_map<std::string, DescHit>();
size_t g_dcache_bytes = 0;
bool dcache_get(const std::string& key, DescHit& out) {
    std::lock_guard<std::mutex> lk(g_dcache_mu);
    auto it = g_dcache.find(key);
    if (it == g_dcache.end()) return false;
    out = it->second;
    return true;
}
void dcache_put(const std::string& key, const DescHit& h) {
    std::lock_guard<std::mutex> lk(g_dcache_mu);
    if (g_dcache_bytes + key.size() > ((size_t)256 << 20)) {
        g_dcache.clear();
        g_dcache_bytes = 0;
    }
    if (g_dcache.emplace(key, h).second) g_dcache_bytes += key.size();
}
}  // namespace

bool jit_compile(const std::string& ptx, std::vector<char>& cubin, std::string& log) {
    nvPTXCompilerHandle h = nullptr;
    if (nvPTXCompilerCreate(&h, ptx.size(), ptx.c_str()) != NVPTXCOMPILE_SUCCESS) {
        log = "nvPTXCompilerCreate failed";
        return false;
    }
    const char* opts[] = {"--gpu-name=sm_100a", "-O3"};
    nvPTXCompileResult rc = nvPTXCompilerCompile(h, 2, opts);
    if (rc != NVPTXCOMPILE_SUCCESS) {
        size_t n = 0;
        nvPTXCompilerGetErrorLogSize(h, &n);
        log.assign(n + 1, '\0');
        if (n) nvPTXCompilerGetErrorLog(h, &log[0]);
        nvPTXCompilerDestroy(&h);
        return false;
    }
    size_t n = 0;
    nvPTXCompilerGetCompiledProgramSize(h, &n);
    cubin.resize(n);
    nvPTXCompilerGetCompiledProgram(h, cubin.data());
    nvPTXCompilerDestroy(&h);
    return true;
}

JitModule::~JitModule() {
    for (Dev& d : dev)
        if (d.lib) cudaLibraryUnload(d.lib);
}

cudaError_t launch_jit(JitKernel& k, const void* P, uint64_t n_tiles, void* psi, uint64_t rank_bits, cudaStream_t st) {
    int dv = 0;
    cudaError_t e = cudaGetDevice(&dv);
    if (e != cudaSuccess) return e;
    JitModule& M = *k.mod;
    std::unique_lock<std::mutex> lk(M.mu);
    if ((int)M.dev.size() <= dv) M.dev.resize(dv + 1);
    JitModule::Dev& D = M.dev[dv];
    if (!D.kern) {
        e = cudaLibraryLoadData(&D.lib, M.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
        if (e != cudaSuccess) return e;
        e = cudaLibraryGetKernel(&D.kern, D.lib, k.name.c_str());
        if (e != cudaSuccess) return e;
        e = cudaKernelSetAttributeForDevice(D.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem, dv);
        if (e != cudaSuccess) return e;
        int sms = 0, occ = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dv);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(D.kern), k.threads,
                                                          k.smem);
        if (e != cudaSuccess) return e;
        static const int occ_cap = std::getenv("QG_DEV_OCC") ? std::atoi(std::getenv("QG_DEV_OCC")) : 0;
        if (occ_cap > 0 && occ > occ_cap) occ = occ_cap;  // dev probe: CTAs per SM cap
        D.grid = sms * (occ > 0 ? occ : 1);
    }
    const uint64_t grid = n_tiles < (uint64_t)D.grid ? n_tiles : (uint64_t)D.grid;
    const cudaKernel_t kern = D.kern;
    lk.unlock();
    void* args[] = {const_cast<void*>(P), &psi, &rank_bits};
    return cudaLaunchKernel(reinterpret_cast<const void*>(kern), dim3((unsigned)grid), dim3(k.threads), args, k.smem,
                            st);
}

// ---------------------------------------------------------------- per-plan compilation
int jit_default_threads() {
    if (const char* e = std::getenv("QG_JIT_THREADS")) {
        const int n = std::atoi(e);
        if (n > 0) return n;
    }
    cpu_set_t cs;
    int n = 0;
    if (sched_getaffinity(0, sizeof cs, &cs) == 0) n = CPU_COUNT(&cs);
    if (n <= 0) n = (int)std::thread::hardware_concurrency();
    return n < 1 ? 1 : (n > 64 ? 64 : n);
}

JitState::~JitState() { join(true); }

void JitState::join(bool cancel) {
    if (cancel) next.store((int64_t)k.size());  // workers stop after their current pass
    for (std::thread& t : workers)
        if (t.joinable()) t.join();
    workers.clear();
}

JitKernel* JitState::try_get(int64_t i) {
    if (i < 0 || i >= (int64_t)k.size()) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (!ready[i]) return nullptr;
    JitKernel* j = k[i].get();
    return (j && j->ok) ? j : nullptr;
}

JitKernel* JitState::wait(int64_t i) {
    if (i < 0 || i >= (int64_t)k.size()) return nullptr;
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return ready[i] != 0; });
    JitKernel* j = k[i].get();
    return (j && j->ok) ? j : nullptr;
}

template <typename Real>
std::shared_ptr<JitState> jit_start(const std::vector<PassDesc<Real>>& d32, int rb, int wb, int nbuf, int threads) {
    auto S = std::make_shared<JitState>();
    const int64_t n = (int64_t)d32.size();
    S->k.resize(n);
    S->ready.assign(n, 0);
    S->t0 = std::chrono::steady_clock::now();
    if (n == 0) return S;
    const PassDesc<Real>* descs = d32.data();
    JitState* st = S.get();
    auto work = [st, descs, n, rb, wb, nbuf]() {
        for (;;) {
            const int64_t i = st->next.fetch_add(1);
            if (i >= n) return;
            const auto c0 = std::chrono::steady_clock::now();
            auto jk = std::make_unique<JitKernel>();
            jk->name = "qg_jit_pass";
            const PassDesc<Real>& P = descs[i];
            // descriptor-keyed level: a pass seen before (same bytes, same kernel shape and
            // variant) reuses its module without re-emitting the PTX
            std::string dkey(reinterpret_cast<const char*>(&P), sizeof(P));
            {
                const int hdr[5] = {(int)sizeof(Real), rb, wb, nbuf, jit_variant()};
                dkey.append(reinterpret_cast<const char*>(hdr), sizeof(hdr));
            }
            DescHit dh;
            if (dcache_get(dkey, dh)) {
                jk->mod = dh.mod;
                jk->smem = dh.smem;
                jk->threads = dh.threads;
                jk->ok = true;
                g_cache_hits.fetch_add(1);
            }
            jk->threads = jk->ok ? jk->threads : jit_block_threads(P, rb, wb, nbuf);
            const std::string ptx = jk->ok ? std::string() : jit_ptx(P, rb, wb, nbuf, jk->name);
            if (jk->ok) {
                // (descriptor cache hit)
            } else if (!ptx.empty()) {
                jk->smem = jit_smem_bytes(P, rb, wb, nbuf);
                if (const char* e = std::getenv("QG_JIT_SMEM_PAD")) jk->smem += (size_t)std::atol(e);  // occupancy probe
                if (auto hit = cache_get(ptx)) {
                    jk->mod = hit;
                    jk->ok = true;
                    g_cache_hits.fetch_add(1);
                } else {
                    auto m = std::make_shared<JitModule>();
                    jk->ok = jit_compile(ptx, m->cubin, jk->err);
                    if (jk->ok) {
                        jk->mod = m;
                        cache_put(ptx, m);
                    }
                }
                if (jk->ok) dcache_put(dkey, DescHit{jk->mod, jk->smem, jk->threads});
            } else {
                jk->err = "pass not covered by the emitter";
            }
            const auto c1 = std::chrono::steady_clock::now();
            st->compile_us += std::chrono::duration_cast<std::chrono::microseconds>(c1 - c0).count();
            (jk->ok ? st->n_ok : st->n_fallback) += 1;
            {
                std::lock_guard<std::mutex> lk(st->mu);
                if (!jk->ok && st->first_error.empty()) st->first_error = jk->err;
                st->k[i] = std::move(jk);
                st->ready[i] = 1;
                st->wall_us = std::chrono::duration_cast<std::chrono::microseconds>(c1 - st->t0).count();
            }
            st->cv.notify_all();
        }
    };
    const int nt = (int)std::min<int64_t>(threads < 1 ? 1 : threads, n);
    for (int t = 0; t < nt; ++t) S->workers.emplace_back(work);
    return S;
}
template std::shared_ptr<JitState> jit_start<float>(const std::vector<PassDesc<float>>&, int, int, int, int);
template std::shared_ptr<JitState> jit_start<double>(const std::vector<PassDesc<double>>&, int, int, int, int);

}  // namespace qg
