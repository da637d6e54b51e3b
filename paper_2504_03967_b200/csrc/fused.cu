// fused.cu — the fused multi-gate pass kernel (sm_100a) and the single-gate kernel.
//
// Replaces the reference's three array kernels (statevec.py:115-144), which
// each stream the whole state through numpy once per gate, with ONE HBM pass
// per group of gates:
//
//   tile   = 2^k amplitudes sharing all index bits outside the pass's tile
//            qubits (desc.tile_q); the 5 lowest tile bits are the lane bits of
//            the io mapping, so global loads/stores are >= 256 B contiguous.
//   thread = 2^RB amplitudes in registers; a register stage applies every op
//            whose target is a register bit with straight-line FMA code
//            (switch over the runtime bit -> compile-time-unrolled body).
//   stage switch = one SMEM round trip with a linear XOR swizzle
//            (conflict-free lanes chosen by the planner).
//   controls / diagonal phases on non-register qubits = per-thread predicates
//            and a per-thread phase accumulator, no data movement.
//
// Memory traffic per pass = read + write of the state once (2 x S bytes),
// the roofline quantity reported by bench.py.
#include <cuda_runtime.h>
#include <stdint.h>

#include "desc.h"
#include "kernels.h"

namespace qg {

static_assert(sizeof(PassDesc<double>) <= 32764, "pass descriptor exceeds the kernel-parameter limit");
static_assert(sizeof(PassDesc<float>) <= 32764, "pass descriptor exceeds the kernel-parameter limit");

template <typename Real>
struct V2;
template <>
struct V2<float> {
    using T = float2;
};
template <>
struct V2<double> {
    using T = double2;
};

// ----------------------------------------------------------------- complex math
// complex64 amplitudes use Blackwell's packed f32x2 FMA/MUL (FFMA2/FMUL2): a
// complex multiply-add by a scalar complex coefficient is two instructions,
// the (im, re) swap and the sign folded into operand modifiers by ptxas.
// complex128 uses scalar DFMA.
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 upk(u64 r) {
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
    u64 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// Operand order matters: data first (ptxas folds the (im, re) swap and the
// partial negate into operand A), coefficient second (scalar broadcast .F32).
// m * x, m = (mr, mi)
__device__ __forceinline__ float2 c_mul(float2 x, float mr, float mi) {
    return upk(fma2(pk(-x.y, x.x), pk(mi, mi), mul2(pk(x.x, x.y), pk(mr, mr))));
}
// acc + m * x
__device__ __forceinline__ float2 c_fma(float2 acc, float2 x, float mr, float mi) {
    return upk(fma2(pk(-x.y, x.x), pk(mi, mi), fma2(pk(x.x, x.y), pk(mr, mr), pk(acc.x, acc.y))));
}
__device__ __forceinline__ float2 r_mul(float2 x, float r) { return upk(mul2(pk(x.x, x.y), pk(r, r))); }
__device__ __forceinline__ float2 r_fma(float2 acc, float2 x, float r) {
    return upk(fma2(pk(x.x, x.y), pk(r, r), pk(acc.x, acc.y)));
}

__device__ __forceinline__ double2 c_mul(double2 x, double mr, double mi) {
    double2 r;
    r.x = mr * x.x - mi * x.y;
    r.y = mr * x.y + mi * x.x;
    return r;
}
__device__ __forceinline__ double2 c_fma(double2 acc, double2 x, double mr, double mi) {
    acc.x += mr * x.x - mi * x.y;
    acc.y += mr * x.y + mi * x.x;
    return acc;
}
__device__ __forceinline__ double2 r_mul(double2 x, double r) {
    x.x *= r;
    x.y *= r;
    return x;
}
__device__ __forceinline__ double2 r_fma(double2 acc, double2 x, double r) {
    acc.x += r * x.x;
    acc.y += r * x.y;
    return acc;
}

template <typename T2>
__device__ __forceinline__ T2 cmul(T2 a, T2 b) {
    return c_mul(a, b.x, b.y);
}

__host__ __device__ constexpr int ctz_c(int x) {  // x in 1..31 (unrolled loop constant)
    return (x & 1) ? 0 : (x & 2) ? 1 : (x & 4) ? 2 : (x & 8) ? 3 : 4;
}
__host__ __device__ constexpr int gray_c(int x) { return x ^ (x >> 1); }

// ----------------------------------------------------------------- register ops
// Every body below is bound to compile-time register bits (TB, CB), so the
// amplitude array never needs runtime indexing; the round loop enables them
// with warp-uniform mask tests (if-then diamonds the register allocator keeps
// in place).
template <int RB, int TB, typename T2, typename Real>
__device__ __forceinline__ void r_dense(T2 (&a)[1 << RB], const Real* __restrict__ m) {
    if constexpr (TB < RB) {
        const Real m00r = m[0], m00i = m[1], m01r = m[2], m01i = m[3];
        const Real m10r = m[4], m10i = m[5], m11r = m[6], m11i = m[7];
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            if (i & (1 << TB)) continue;
            const int j = i | (1 << TB);
            const T2 x = a[i], y = a[j];
            a[i] = c_fma(c_mul(x, m00r, m00i), y, m01r, m01i);
            a[j] = c_fma(c_mul(x, m10r, m10i), y, m11r, m11i);
        }
    }
}

// real 2x2 (H, RY and their products): half the work of the complex case
template <int RB, int TB, typename T2, typename Real>
__device__ __forceinline__ void r_rdense(T2 (&a)[1 << RB], const Real* __restrict__ m) {
    if constexpr (TB < RB) {
        const Real m00 = m[0], m01 = m[1], m10 = m[2], m11 = m[3];
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            if (i & (1 << TB)) continue;
            const int j = i | (1 << TB);
            const T2 x = a[i], y = a[j];
            a[i] = r_fma(r_mul(x, m00), y, m01);
            a[j] = r_fma(r_mul(x, m10), y, m11);
        }
    }
}

template <int RB, int TB, typename T2>
__device__ __forceinline__ void r_diag(T2 (&a)[1 << RB], T2 d0, T2 d1, bool lo_id) {
    if constexpr (TB < RB) {
        if (lo_id) {
#pragma unroll
            for (int i = 0; i < (1 << RB); ++i)
                if (i & (1 << TB)) a[i] = cmul(a[i], d1);
        } else {
#pragma unroll
            for (int i = 0; i < (1 << RB); ++i) a[i] = cmul(a[i], (i & (1 << TB)) ? d1 : d0);
        }
    }
}

template <int RB, int TB, typename T2>
__device__ __forceinline__ void r_x(T2 (&a)[1 << RB]) {
    if constexpr (TB < RB) {
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            if (i & (1 << TB)) continue;
            const T2 x = a[i];
            a[i] = a[i | (1 << TB)];
            a[i | (1 << TB)] = x;
        }
    }
}

template <int RB, int TB, int CB, typename T2>
__device__ __forceinline__ void r_cx(T2 (&a)[1 << RB]) {
    if constexpr (TB < RB && CB < RB && TB != CB) {
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            if ((i & (1 << TB)) || !(i & (1 << CB))) continue;
            const T2 x = a[i];
            a[i] = a[i | (1 << TB)];
            a[i | (1 << TB)] = x;
        }
    }
}

template <int RB, int TB, int CB, typename T2>
__device__ __forceinline__ void r_cphase(T2 (&a)[1 << RB], T2 e) {
    if constexpr (TB < RB && CB < RB && TB != CB) {
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i)
            if ((i & (1 << TB)) && (i & (1 << CB))) a[i] = cmul(a[i], e);
    }
}

// CPHASE when the thread's register flips move the |11> quadrant to (1^ft, 1^fc)
template <int RB, int TB, int CB, typename T2>
__device__ __forceinline__ void r_cphase_flip(T2 (&a)[1 << RB], T2 e, uint32_t ft, uint32_t fc) {
    if constexpr (TB < RB && CB < RB && TB != CB) {
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            const uint32_t bt = ((i >> TB) & 1) ^ ft, bc = ((i >> CB) & 1) ^ fc;
            T2 v;
            v.x = (bt & bc) ? e.x : decltype(e.x)(1);
            v.y = (bt & bc) ? e.y : decltype(e.y)(0);
            a[i] = cmul(a[i], v);
        }
    }
}

// select between a and b without branching (per-thread condition)
template <typename Real>
__device__ __forceinline__ Real sel(bool c, Real a, Real b) { return c ? a : b; }

// One round: slots in the fixed order dense < cdiag < diag < X < CX < CPHASE (desc.h).
// F is the thread's register flip mask: register slot i holds the amplitude of
// logical register index i ^ F (X ops under thread-level controls only toggle
// F; the next transpose / store writes through the flipped addresses).
template <int RB, typename T2, typename Real>
__device__ __forceinline__ void run_round(T2 (&a)[1 << RB], const PassDesc<Real>& P, const RoundDesc& R, uint64_t tb,
                                          uint32_t& F) {
    int ci = R.coef;
    int ei = R.ent;
    const uint32_t md = R.dense, mr = R.rdense;
    if (md | mr) {
        // flipped bit: X U X = U with rows and columns swapped
#define QG_DENSE(B)                                                                      \
    if (B < RB) {                                                                        \
        if (md & (1u << B)) {                                                            \
            const Real* m = P.coef[ci];                                                  \
            const bool f = (F >> B) & 1u;                                                \
            Real c[8];                                                                   \
            c[0] = sel(f, m[6], m[0]); c[1] = sel(f, m[7], m[1]);                        \
            c[2] = sel(f, m[4], m[2]); c[3] = sel(f, m[5], m[3]);                        \
            c[4] = sel(f, m[2], m[4]); c[5] = sel(f, m[3], m[5]);                        \
            c[6] = sel(f, m[0], m[6]); c[7] = sel(f, m[1], m[7]);                        \
            r_dense<RB, B>(a, c);                                                        \
            ++ci;                                                                        \
        }                                                                                \
        if (mr & (1u << B)) {                                                            \
            const Real* m = P.coef[ci];                                                  \
            const bool f = (F >> B) & 1u;                                                \
            Real c[4];                                                                   \
            c[0] = sel(f, m[3], m[0]); c[1] = sel(f, m[2], m[1]);                        \
            c[2] = sel(f, m[1], m[2]); c[3] = sel(f, m[0], m[3]);                        \
            r_rdense<RB, B>(a, c);                                                       \
            ++ci;                                                                        \
        }                                                                                \
    }
        QG_DENSE(0) QG_DENSE(1) QG_DENSE(2) QG_DENSE(3) QG_DENSE(4)
#undef QG_DENSE
    }
    const uint32_t mk = R.cdiag;
    if (mk) {
#define QG_CDIAG(B)                                                                      \
    if (B < RB && (mk & (1u << B))) {                                                    \
        const Real* m = P.coef[ci];                                                      \
        ++ci;                                                                            \
        const bool f = (F >> B) & 1u;                                                    \
        T2 d0, d1;                                                                       \
        d0.x = sel(f, m[2], m[0]); d0.y = sel(f, m[3], m[1]);                            \
        d1.x = sel(f, m[0], m[2]); d1.y = sel(f, m[1], m[3]);                            \
        r_diag<RB, B>(a, d0, d1, false);                                                 \
    }
        QG_CDIAG(0) QG_CDIAG(1) QG_CDIAG(2) QG_CDIAG(3) QG_CDIAG(4)
#undef QG_CDIAG
    }
    const uint32_t mg = R.diag;
    if (mg) {
        const uint32_t mh = R.dhi;
#define QG_DIAG(B)                                                                       \
    if (B < RB && (mg & (1u << B))) {                                                    \
        T2 d0, d1;                                                                       \
        d0.x = Real(1); d0.y = Real(0); d1 = d0;                                         \
        const int ne = R.dcnt[B];                                                        \
        for (int e = 0; e < ne; ++e, ++ei) {                                             \
            const Entry<Real>& E = P.ent[ei];                                            \
            if ((tb & E.cmask) != E.cmask) continue;                                     \
            T2 v0, v1;                                                                   \
            v0.x = E.v[0]; v0.y = E.v[1]; v1.x = E.v[2]; v1.y = E.v[3];                  \
            d0 = cmul(d0, v0);                                                           \
            d1 = cmul(d1, v1);                                                           \
        }                                                                                \
        const bool f = (F >> B) & 1u;                                                    \
        if ((mh & (1u << B)) && !f) {                                                    \
            r_diag<RB, B>(a, d0, d1, true);                                              \
        } else {                                                                         \
            T2 e0, e1;                                                                   \
            e0.x = sel(f, d1.x, d0.x); e0.y = sel(f, d1.y, d0.y);                        \
            e1.x = sel(f, d0.x, d1.x); e1.y = sel(f, d0.y, d1.y);                        \
            r_diag<RB, B>(a, e0, e1, false);                                             \
        }                                                                                \
    }
        QG_DIAG(0) QG_DIAG(1) QG_DIAG(2) QG_DIAG(3) QG_DIAG(4)
#undef QG_DIAG
    }
    const uint32_t mx = R.xs;
    if (mx) {
#define QG_X(B)                                                                          \
    if (B < RB && (mx & (1u << B))) {                                                    \
        uint32_t odd = 0;                                                                \
        const int ne = R.xcnt[B];                                                        \
        for (int e = 0; e < ne; ++e, ++ei) {                                             \
            const uint64_t cm = P.ent[ei].cmask;                                         \
            odd ^= (tb & cm) == cm ? 1u : 0u;                                            \
        }                                                                                \
        F ^= odd << B;                                                                   \
    }
        QG_X(0) QG_X(1) QG_X(2) QG_X(3) QG_X(4)
#undef QG_X
    }
    uint32_t mc = R.cx;
    // iterate over the set CX slots in (t, c) order; one switch case per slot keeps
    // every body a real branch (if-converted bodies would all be issued predicated)
    while (mc) {
        const int k = __ffs(mc) - 1;
        mc &= mc - 1;
        switch (k) {
#define QG_CXK(T, C)                                                                     \
    case 5 * T + C:                                                                      \
        if constexpr (T < RB && C < RB && T != C) {                                      \
            r_cx<RB, T, C>(a);                                                           \
            F ^= ((F >> C) & 1u) << T;                                                   \
        }                                                                                \
        break;
#define QG_CXT(T) QG_CXK(T, 0) QG_CXK(T, 1) QG_CXK(T, 2) QG_CXK(T, 3) QG_CXK(T, 4)
            QG_CXT(0) QG_CXT(1) QG_CXT(2) QG_CXT(3) QG_CXT(4)
#undef QG_CXT
#undef QG_CXK
            default: break;
        }
    }
    const uint32_t mp = R.cp;
    if (mp) {
        // flipped bits move the phased quadrant: use the general 4-quadrant form then
#define QG_CP(T, C)                                                                      \
    if (T < RB && (mp & (1u << (T * (T - 1) / 2 + C)))) {                                \
        T2 e;                                                                            \
        e.x = P.coef[ci][0]; e.y = P.coef[ci][1]; ++ci;                                  \
        if (((F >> T) | (F >> C)) & 1u) r_cphase_flip<RB, T, C>(a, e, (F >> T) & 1u, (F >> C) & 1u); \
        else r_cphase<RB, T, C>(a, e);                                                   \
    }
        QG_CP(1, 0) QG_CP(2, 0) QG_CP(2, 1) QG_CP(3, 0) QG_CP(3, 1) QG_CP(3, 2)
        QG_CP(4, 0) QG_CP(4, 1) QG_CP(4, 2) QG_CP(4, 3)
#undef QG_CP
    }
}

// ----------------------------------------------------------------- mappings
template <int WB>
__device__ __forceinline__ uint64_t thread_gbits(const StageDesc& S, int lane, int warp) {
    uint64_t g = 0;
#pragma unroll
    for (int l = 0; l < kLaneBits; ++l) g |= (uint64_t)((lane >> l) & 1) << S.lane_q[l];
#pragma unroll
    for (int w = 0; w < WB; ++w) g |= (uint64_t)((warp >> w) & 1) << S.warp_q[w];
    return g;
}

template <int WB>
__device__ __forceinline__ uint32_t thread_soff(const StageDesc& S, int lane, int warp) {
    uint32_t s = 0;
#pragma unroll
    for (int l = 0; l < kLaneBits; ++l) s ^= ((lane >> l) & 1) ? (uint32_t)S.lane_s[l] : 0u;
#pragma unroll
    for (int w = 0; w < WB; ++w) s ^= ((warp >> w) & 1) ? (uint32_t)S.warp_s[w] : 0u;
    return s;
}

// SMEM offsets are kept in BYTES (swizzled amplitude index * sizeof(T2)) so an
// access is one LOP3 (xor) + STS/LDS [reg + smem_base] with no scaling.
template <int RB, typename T2>
__device__ __forceinline__ void smem_put(char* sm, const StageDesc& S, uint32_t so, const T2 (&a)[1 << RB],
                                         uint32_t F) {
    constexpr int sh = sizeof(T2) == 8 ? 3 : 4;
    uint32_t rs[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) rs[b] = (uint32_t)S.out_s[b] << sh;
#pragma unroll
    for (int b = 0; b < RB; ++b)
        if ((F >> b) & 1u) so ^= rs[b];
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (j) so ^= rs[ctz_c(j)];
        *reinterpret_cast<T2*>(sm + so) = a[gray_c(j)];
    }
}

template <int RB, typename T2>
__device__ __forceinline__ void smem_get(const char* sm, const StageDesc& S, uint32_t so, T2 (&a)[1 << RB]) {
    constexpr int sh = sizeof(T2) == 8 ? 3 : 4;
    uint32_t rs[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) rs[b] = (uint32_t)S.reg_s[b] << sh;
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (j) so ^= rs[ctz_c(j)];
        a[gray_c(j)] = *reinterpret_cast<const T2*>(sm + so);
    }
}

// ----------------------------------------------------------------- the kernel
// Dynamic SMEM layout: [2 tile buffers: 2 x 2^k amplitudes, used alternately so
// a transpose needs one barrier] [tile-id -> base index tables:
// 4 x 256 u64] [per mapping m (io + stages): lane -> global bits (32 u64),
// warp -> global bits (16 u64), lane -> SMEM byte offset (32 u32), warp -> SMEM
// byte offset (16 u32)].  The tables are built once per CTA, so per tile and
// per stage a thread's index bits cost a few LDS instead of bit-deposit loops.
constexpr int kMapG = 48;   // u64 entries per mapping (32 lanes + 16 warps)
constexpr int kMapS = 48;   // u32 entries per mapping
__host__ __device__ constexpr size_t tables_bytes() {
    return 4 * 256 * 8 + (kMaxStages + 1) * (kMapG * 8 + kMapS * 4);
}

template <typename Real, int RB, int WB>
__global__ void __launch_bounds__(32 << WB, (WB >= 4 || sizeof(Real) == 8) ? 1 : 2)
    fused_pass_kernel(const __grid_constant__ PassDesc<Real> P, typename V2<Real>::T* __restrict__ psi,
                      uint64_t rank_bits) {
    using T2 = typename V2<Real>::T;
    constexpr int R = 1 << RB;
    constexpr int NT = 32 << WB;
    constexpr int sh = sizeof(T2) == 8 ? 3 : 4;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    char* sm = reinterpret_cast<char*>(smem_raw);
    const int k = P.k;
    const uint32_t buf_bytes = (uint32_t)sizeof(T2) << k;
    uint64_t* tbase = reinterpret_cast<uint64_t*>(smem_raw + 2 * (size_t)buf_bytes);
    uint64_t* tmg = tbase + 4 * 256;
    uint32_t* tms = reinterpret_cast<uint32_t*>(tmg + (kMaxStages + 1) * kMapG);
    const int ns = P.n_stages;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;

    // ---- per-CTA tables
    const int n_comp = 64 - __clzll((long long)P.n_tiles) - 1;  // tile-id bits
    for (int e = tid; e < 4 * 256; e += NT) {
        const int t = e >> 8, v = e & 255;
        uint64_t g = 0;
        for (int j = 0; j < 8; ++j)
            if (((v >> j) & 1) && 8 * t + j < n_comp) g |= 1ull << P.comp_q[8 * t + j];
        tbase[e] = g;
    }
    for (int e = tid; e < (ns + 1) * kMapG; e += NT) {
        const int m = e / kMapG, x = e % kMapG;
        const StageDesc& S = P.stg[m];
        uint64_t g = 0;
        uint32_t so = 0;
        if (x < 32) {
            for (int l = 0; l < kLaneBits; ++l)
                if ((x >> l) & 1) { g |= 1ull << S.lane_q[l]; so ^= S.lane_s[l]; }
        } else {
            for (int w = 0; w < WB; ++w)
                if (((x - 32) >> w) & 1) { g |= 1ull << S.warp_q[w]; so ^= S.warp_s[w]; }
        }
        tmg[e] = g;
        tms[e] = so << sh;
    }
    __syncthreads();

    const int li = P.load_direct ? 1 : 0;   // mapping used for the global load
    const int si = P.store_direct ? ns : 0; // mapping used for the global store
    auto tgb = [&](int m) { return tmg[m * kMapG + lane] | tmg[m * kMapG + 32 + warp]; };
    auto tso = [&](int m) { return tms[m * kMapS + lane] ^ tms[m * kMapS + 32 + warp]; };
    T2 a[R];
    uint32_t buf = 0;  // byte offset of the tile buffer the next transpose writes

    for (uint64_t tile = blockIdx.x; tile < P.n_tiles; tile += gridDim.x) {
        const uint64_t base = tbase[tile & 255] | tbase[256 + ((tile >> 8) & 255)] |
                              tbase[512 + ((tile >> 16) & 255)] | tbase[768 + ((tile >> 24) & 255)];
        {  // global load, Gray-code order over the register index
            const StageDesc& S = P.stg[li];
            uint64_t g = base | tgb(li);
#pragma unroll
            for (int j = 0; j < R; ++j) {
                if (j) g ^= 1ull << S.reg_q[ctz_c(j)];
                a[gray_c(j)] = __ldcs(psi + g);
            }
        }
        int cur = li;
        uint32_t F = 0;  // register flip mask (see run_round)
        for (int s = 1; s <= ns; ++s) {
            const StageDesc& S = P.stg[s];
            if (cur != s) {  // SMEM transpose into this stage's mapping
                smem_put<RB>(sm + buf, P.stg[cur], tso(cur), a, F);
                __syncthreads();
                smem_get<RB>(sm + buf, S, tso(s), a);
                buf ^= buf_bytes;
                cur = s;
                F = 0;
            }
            const uint64_t tb = base | rank_bits | tgb(s);
            for (int r = S.round_begin; r < S.round_end; ++r) run_round<RB>(a, P, P.rounds[r], tb, F);
            if (S.tph_end > S.tph_begin) {  // thread-level phases commute with the whole stage
                T2 ph;
                ph.x = Real(1);
                ph.y = Real(0);
                for (int e = S.tph_begin; e < S.tph_end; ++e) {
                    const Entry<Real>& E = P.ent[e];
                    if ((tb & E.cmask) != E.cmask) continue;
                    const bool hi = (tb & E.qmask) != 0;
                    T2 v;
                    v.x = hi ? E.v[2] : E.v[0];
                    v.y = hi ? E.v[3] : E.v[1];
                    ph = cmul(ph, v);
                }
#pragma unroll
                for (int i = 0; i < R; ++i) a[i] = cmul(a[i], ph);
            }
        }
        if (cur != si) {
            smem_put<RB>(sm + buf, P.stg[cur], tso(cur), a, F);
            __syncthreads();
            smem_get<RB>(sm + buf, P.stg[si], tso(si), a);
            buf ^= buf_bytes;
            F = 0;
        }
        {  // global store through the output mapping (deferred CX + flips folded in)
            const StageDesc& S = P.stg[si];
            uint64_t og[RB];
#pragma unroll
            for (int b = 0; b < RB; ++b) og[b] = S.out_g[b];
            uint64_t g = base | tgb(si);
#pragma unroll
            for (int b = 0; b < RB; ++b)
                if ((F >> b) & 1u) g ^= og[b];
#pragma unroll
            for (int j = 0; j < R; ++j) {
                if (j) g ^= og[ctz_c(j)];
                __stcs(psi + g, a[gray_c(j)]);
            }
        }
    }
}

// ----------------------------------------------------------------- single-gate kernel
template <typename Real>
__global__ void gate_kernel(typename V2<Real>::T* __restrict__ psi, int n_local, GateOp op, uint64_t rank_bits) {
    using T2 = typename V2<Real>::T;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    if (op.kind == 0) {
        const int t = op.t;
        const uint64_t npairs = 1ull << (n_local - 1);
        const Real m00r = (Real)op.m[0], m00i = (Real)op.m[1], m01r = (Real)op.m[2], m01i = (Real)op.m[3];
        const Real m10r = (Real)op.m[4], m10i = (Real)op.m[5], m11r = (Real)op.m[6], m11i = (Real)op.m[7];
        for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npairs; p += stride) {
            const uint64_t i0 = ((p >> t) << (t + 1)) | (p & ((1ull << t) - 1ull));
            const uint64_t i1 = i0 | (1ull << t);
            if (((rank_bits | i0) & op.cmask) != op.cmask) continue;
            const T2 x = psi[i0], y = psi[i1];
            T2 u, v;
            u.x = m00r * x.x - m00i * x.y + m01r * y.x - m01i * y.y;
            u.y = m00r * x.y + m00i * x.x + m01r * y.y + m01i * y.x;
            v.x = m10r * x.x - m10i * x.y + m11r * y.x - m11i * y.y;
            v.y = m10r * x.y + m10i * x.x + m11r * y.y + m11i * y.x;
            psi[i0] = u;
            psi[i1] = v;
        }
    } else {
        const uint64_t namps = 1ull << n_local;
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < namps; i += stride) {
            const uint64_t g = rank_bits | i;
            if ((g & op.cmask) != op.cmask) continue;
            const bool hi = (g & op.qmask) != 0;
            T2 v;
            v.x = (Real)(hi ? op.m[2] : op.m[0]);
            v.y = (Real)(hi ? op.m[3] : op.m[1]);
            psi[i] = cmul(psi[i], v);
        }
    }
}

// ----------------------------------------------------------------- launchers
template <typename Real, int RB, int WB>
static cudaError_t launch_fused_t(const PassDesc<Real>& P, void* psi, uint64_t rank_bits, cudaStream_t st) {
    constexpr int threads = 32 << WB;
    const int k = RB + kLaneBits + WB;
    const size_t smem = 2 * ((size_t)1 << k) * sizeof(typename V2<Real>::T) + tables_bytes();
    auto kern = fused_pass_kernel<Real, RB, WB>;
    static int max_blocks = -1;  // per instantiation: resident CTAs per SM x SMs
    if (max_blocks < 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        if (e != cudaSuccess) return e;
        max_blocks = sms * (occ > 0 ? occ : 1);
    }
    const uint64_t grid = P.n_tiles < (uint64_t)max_blocks ? P.n_tiles : (uint64_t)max_blocks;
    kern<<<(unsigned)grid, threads, smem, st>>>(P, reinterpret_cast<typename V2<Real>::T*>(psi), rank_bits);
    return cudaGetLastError();
}

cudaError_t launch_fused(int dtype, int cfg_id, const void* desc, void* psi, uint64_t rank_bits, cudaStream_t st) {
    // must match kCfgC64 / kCfgC128 in plan.cpp
    if (dtype == 0) {
        const auto& P = *static_cast<const PassDesc<float>*>(desc);
        switch (cfg_id) {
            case 0: return launch_fused_t<float, 4, 4>(P, psi, rank_bits, st);
            case 1: return launch_fused_t<float, 4, 3>(P, psi, rank_bits, st);
            case 2: return launch_fused_t<float, 4, 2>(P, psi, rank_bits, st);
            default: return launch_fused_t<float, 3, 0>(P, psi, rank_bits, st);
        }
    }
    const auto& P = *static_cast<const PassDesc<double>*>(desc);
    switch (cfg_id) {
        case 0: return launch_fused_t<double, 4, 3>(P, psi, rank_bits, st);
        case 1: return launch_fused_t<double, 3, 2>(P, psi, rank_bits, st);
        default: return launch_fused_t<double, 3, 0>(P, psi, rank_bits, st);
    }
}

cudaError_t launch_gate(int dtype, const GateOp& op, void* psi, int n_local, uint64_t rank_bits, cudaStream_t st) {
    const uint64_t work = op.kind == 0 ? (1ull << (n_local - 1)) : (1ull << n_local);
    const int threads = 256;
    uint64_t blocks = (work + threads - 1) / threads;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    if (dtype == 0)
        gate_kernel<float><<<(unsigned)blocks, threads, 0, st>>>(static_cast<float2*>(psi), n_local, op, rank_bits);
    else
        gate_kernel<double><<<(unsigned)blocks, threads, 0, st>>>(static_cast<double2*>(psi), n_local, op, rank_bits);
    return cudaGetLastError();
}

}  // namespace qg
