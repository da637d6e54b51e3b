// fused.cu — the fused multi-gate pass kernel (sm_100a) and the single-gate kernel.
//
// Replaces the reference's three array kernels (statevec.py:115-144), which
// each stream the whole state through numpy once per gate, with ONE HBM pass
// per group of gates:
//
//   tile   = 2^k amplitudes sharing all index bits outside the pass's tile
//            qubits (desc.tile_q); the 5 lowest tile bits are the lane bits of
//            the io mapping, so global loads/stores are >= 256 B contiguous.
//   thread = 2^RB amplitudes in registers ("slots"); a register stage runs its
//            op list (desc.h): each 32-bit op word is dispatched through a PTX
//            jump table to a body whose slot bits are compile-time constants,
//            so the slot array is only indexed by constants (straight-line
//            packed-f32x2 FMA code).
//   lazy CX = register CX gates never touch data: the planner tracks the GF(2)
//            map L (slot p holds logical index L^-1 (p ^ F)) and the transpose /
//            store addresses apply it at the stage end.
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
#include "jt_lists.h"
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
__device__ __forceinline__ double2 r_fma(double2 acc, double2 x, double r) {
    acc.x += r * x.x;
    acc.y += r * x.y;
    return acc;
}

template <typename T2>
__device__ __forceinline__ T2 cmul(T2 a, T2 b) {
    return c_mul(a, b.x, b.y);
}

__host__ __device__ constexpr int ctz_c(int x) {  // x in 1..63 (unrolled loop constant)
    return (x & 1) ? 0 : (x & 2) ? 1 : (x & 4) ? 2 : (x & 8) ? 3 : (x & 16) ? 4 : 5;
}
static_assert(ctz_c(32) == 5 && ctz_c(48) == 4 && ctz_c(8) == 3, "ctz_c");
__host__ __device__ constexpr int gray_c(int x) { return x ^ (x >> 1); }

// ----------------------------------------------------------------- register ops
// Every body below is bound to compile-time slot vectors (V, W, TB, CB), so the
// amplitude array is never indexed at run time: after unrolling, each body is
// straight-line FMA code on fixed registers.
__host__ __device__ constexpr int parity_c(uint32_t x) {
    x ^= x >> 16; x ^= x >> 8; x ^= x >> 4; x ^= x >> 2; x ^= x >> 1;
    return (int)(x & 1u);
}

// complex 2x2 on pairs {i, i ^ V}, i the member with parity(W & i) = 0
template <int RB, uint32_t V, uint32_t W, typename T2, typename Real>
__device__ __forceinline__ void p_dense(T2 (&a)[1 << RB], const Real* __restrict__ m) {
    const Real m00r = m[0], m00i = m[1], m01r = m[2], m01i = m[3];
    const Real m10r = m[4], m10i = m[5], m11r = m[6], m11i = m[7];
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) {
        if (parity_c(W & (uint32_t)i)) continue;
        const int j = i ^ (int)V;
        // each output's final FMA is the last use of its own input, so the
        // allocator writes it in place (no copies back into the array registers)
        const T2 x = a[i], y = a[j];
        const T2 ty = c_mul(y, m01r, m01i), tx = c_mul(x, m10r, m10i);
        a[i] = c_fma(ty, x, m00r, m00i);
        a[j] = c_fma(tx, y, m11r, m11i);
    }
}

// rotation by shears on pairs {i, i ^ V} (x = the parity(W & i) = 0 member):
// x += a y; y += b x; x += a y — every FMA updates its own register in place
template <int RB, uint32_t V, uint32_t W, typename T2, typename Real>
__device__ __forceinline__ void p_rot(T2 (&a)[1 << RB], Real sa, Real sb) {
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) {
        if (parity_c(W & (uint32_t)i)) continue;
        const int j = i ^ (int)V;
        a[i] = r_fma(a[i], a[j], sa);
    }
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) {
        if (parity_c(W & (uint32_t)i)) continue;
        const int j = i ^ (int)V;
        a[j] = r_fma(a[j], a[i], sb);
    }
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) {
        if (parity_c(W & (uint32_t)i)) continue;
        const int j = i ^ (int)V;
        a[i] = r_fma(a[i], a[j], sa);
    }
}

// x e on the slots with parity(W & i) == P
template <int RB, uint32_t W, int P, typename T2>
__device__ __forceinline__ void p_phase(T2 (&a)[1 << RB], T2 e) {
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i)
        if (parity_c(W & (uint32_t)i) == P) a[i] = cmul(a[i], e);
}

// x d0 / d1 on the slots with parity(W & i) == 0 / 1
template <int RB, uint32_t W, typename T2>
__device__ __forceinline__ void p_diag(T2 (&a)[1 << RB], T2 d0, T2 d1) {
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) a[i] = cmul(a[i], parity_c(W & (uint32_t)i) ? d1 : d0);
}

// value copy through the FP pipe (x * 1): opaque to the register allocator's copy
// coalescing, so a permuting body writes its results into the loop-carried
// registers like any arithmetic body (plain moves make ptxas copy the whole
// amplitude array at the op loop head)
__device__ __forceinline__ float2 ocopy(float2 x) { return upk(mul2(pk(x.x, x.y), pk(1.0f, 1.0f))); }
__device__ __forceinline__ double2 ocopy(double2 x) {
    double2 r;
    asm("mul.rn.f64 %0, %1, 0d3FF0000000000000;" : "=d"(r.x) : "d"(x.x));
    asm("mul.rn.f64 %0, %1, 0d3FF0000000000000;" : "=d"(r.y) : "d"(x.y));
    return r;
}

template <int RB, int TB, int CB, typename T2>
__device__ __forceinline__ void r_cx(T2 (&a)[1 << RB]) {
    if constexpr (TB < RB && CB < RB && TB != CB) {
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            if ((i & (1 << TB)) || !(i & (1 << CB))) continue;
            const T2 x = ocopy(a[i]);
            a[i] = ocopy(a[i | (1 << TB)]);
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

// CPHASE when the thread's flips move the |11> quadrant to (1^ft, 1^fc)
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

// Thread predicate of an op: every global-index bit of the mask is 1 for this thread.
__device__ __forceinline__ bool pred_ok(uint64_t tb, uint64_t m) { return (tb & m) == m; }

// pair-op bodies: flip-select the coefficients (X U X when the thread's roles
// are swapped), then run the compile-time body
// rotation R(psi) as three in-place shears (planner: Emitter::rotation); a thread
// whose roles are swapped sees X R X = R(-psi): both shear coefficients negate
// complex64: the scaled two-FMA form (planner: Emitter::rotation), m = (k, form):
//   form 0: x' = x - k y, y' = y + k x        form 1: x' = k x - y, y' = x + k y
// (R(psi) / sigma; the pass applies sigma's product once at its end).  Swapped roles see
// R(-psi) / sigma: form 0 with -k, form 1 with the unit terms negated.
// Every output is one fmaf of the inputs, as the JIT kernels compute it (bit-identical).
template <int RB, uint32_t V, uint32_t W>
__device__ __forceinline__ void p_rot_scaled(float2 (&a)[1 << RB], float k, float form, bool f) {
    if (form == 0.0f) {
        const float kk = f ? -k : k, nk = -kk;
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            if (parity_c(W & (uint32_t)i)) continue;
            const int j = i ^ (int)V;
            const float2 x = a[i], y = a[j];
            a[i] = make_float2(fmaf(y.x, nk, x.x), fmaf(y.y, nk, x.y));
            a[j] = make_float2(fmaf(x.x, kk, y.x), fmaf(x.y, kk, y.y));
        }
    } else if (!f) {
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            if (parity_c(W & (uint32_t)i)) continue;
            const int j = i ^ (int)V;
            const float2 x = a[i], y = a[j];
            a[i] = make_float2(fmaf(x.x, k, -y.x), fmaf(x.y, k, -y.y));
            a[j] = make_float2(fmaf(y.x, k, x.x), fmaf(y.y, k, x.y));
        }
    } else {  // swapped roles: the unit terms negate
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            if (parity_c(W & (uint32_t)i)) continue;
            const int j = i ^ (int)V;
            const float2 x = a[i], y = a[j];
            a[i] = make_float2(fmaf(x.x, k, y.x), fmaf(x.y, k, y.y));
            a[j] = make_float2(fmaf(y.x, k, -x.x), fmaf(y.y, k, -x.y));
        }
    }
}
template <int RB, uint32_t V, uint32_t W, typename T2, typename Real>
__device__ __forceinline__ void op_rd(T2 (&a)[1 << RB], const Real* m, uint32_t F) {
    const bool f = parity_c(W & F);
    if constexpr (sizeof(Real) == 4) {
        p_rot_scaled<RB, V, W>(a, m[0], m[1], f);
    } else {
        const Real sa = sel(f, -m[0], m[0]), sb = sel(f, -m[1], m[1]);
        p_rot<RB, V, W>(a, sa, sb);
    }
}
template <int RB, uint32_t V, uint32_t W, typename T2, typename Real>
__device__ __forceinline__ void op_cd(T2 (&a)[1 << RB], const Real* m, uint32_t F) {
    const bool f = parity_c(W & F);
    Real c[8];
    c[0] = sel(f, m[6], m[0]); c[1] = sel(f, m[7], m[1]);
    c[2] = sel(f, m[4], m[2]); c[3] = sel(f, m[5], m[3]);
    c[4] = sel(f, m[2], m[4]); c[5] = sel(f, m[3], m[5]);
    c[6] = sel(f, m[0], m[6]); c[7] = sel(f, m[1], m[7]);
    p_dense<RB, V, W>(a, c);
}
// x e on logical |1> = slots with parity(W & p) ^ f = 1; warp-uniform f takes the
// half-multiply path (1 complex multiply per 2 amplitudes)
template <int RB, uint32_t W, typename T2, typename Real>
__device__ __forceinline__ void op_ph(T2 (&a)[1 << RB], T2 e, uint32_t F) {
    const bool f = parity_c(W & F);
    const uint32_t bal = __ballot_sync(0xffffffffu, f);
    if (bal == 0u) {
        p_phase<RB, W, 1>(a, e);
    } else if (bal == 0xffffffffu) {
        p_phase<RB, W, 0>(a, e);
    } else {
        T2 d0, d1;
        d0.x = sel(f, e.x, Real(1)); d0.y = sel(f, e.y, Real(0));
        d1.x = sel(f, Real(1), e.x); d1.y = sel(f, Real(0), e.y);
        p_diag<RB, W>(a, d0, d1);
    }
}

// the thread's phase of an OC_PH word: product of its list entries whose
// predicate holds (e.g. all the CR1 gates of a QFT row sharing one register target)
template <bool UPH, typename T2, typename Real>
__device__ __forceinline__ T2 ph_product(const PassDesc<Real>& P, uint32_t w, uint64_t tb) {
    const int n = (w >> 8) & 0x7fu, b = w >> 16;
    T2 e;  // entry 0 is the unconditional factor (planner: emit_group)
    e.x = P.ph[b].e[0];
    e.y = P.ph[b].e[1];
    if constexpr (UPH) {  // passes with tile-uniform slots (the kernel variant that computes them)
        if (w & 0x8000u) {  // the tile-uniform factors, computed at the tile start (slot in entry 0's pad)
            extern __shared__ __align__(16) unsigned char smem_raw[];
            e = cmul(e, reinterpret_cast<const T2*>(smem_raw)[P.ph[b].pad]);
        }
    }
    for (int k = 1; k < n; ++k) {
        const PhEnt<Real>& E = P.ph[b + k];
        const bool on = (tb >> E.pos) & 1u;
        T2 v;
        v.x = on ? E.e[0] : Real(1);
        v.y = on ? E.e[1] : Real(0);
        e = cmul(e, v);
    }
    return e;
}

// One op word (desc.h).  F is the thread's flip vector: slot p holds logical
// register index L^-1 (p ^ F).  Case labels are the dense codes of desc.h for
// this RB; bodies that do not exist for this RB get unique unreachable labels.
//
// Dispatch: NVVM lowers this switch to a compare tree (~7 dependent ISETP+BRA
// levels per op, the largest single overhead of the interpreter).  With
// QG_JT the switch is entered through a PTX jump table instead: `brx.idx` on
// the body code (ptxas emits one BRX and drops the then-unreachable tree), its
// targets being PTX labels placed as the first statement of every case.  The
// labels re-define the live values (w, tb, F) so everything a body computes
// sits after its label; build.py verifies in the PTX that each label starts its
// basic block and rebuilds without QG_JT otherwise.
#ifndef QG_NO_JT
#define QG_JT 1
#endif
#ifdef QG_JT
#define QGJ_ENTER(name) asm volatile(name ":" ::: "memory")
#else
#define QGJ_ENTER(name) ((void)0)
#endif
#define QG_LAB(ok, code, junk) ((ok) ? (code) : 1000 + (junk))
template <int RB, bool UPH, typename T2, typename Real>
__device__ __forceinline__ void run_stage_ops(T2 (&a)[1 << RB], const PassDesc<Real>& P, int o, uint64_t tb,
                                              uint32_t& F) {
    // op words are read through a running byte offset (no per-op index math) and
    // one word ahead; the list ends with an OC_END word (no per-op bound check)
    const char* opb = reinterpret_cast<const char*>(P.ops);
    uint32_t ob = (uint32_t)o * 4u;
    uint32_t w = *reinterpret_cast<const uint32_t*>(opb + ob);
  for (;;) {
    ob += 4u;
    const uint32_t wn = *reinterpret_cast<const uint32_t*>(opb + ob);
#ifdef QG_JT
    {
        const uint32_t code = w & 0xffu;
        if constexpr (RB == 6) {
            static_assert(QGJ_N_6 == oc_xf(6), "jt_lists.h out of date");
            const uint32_t idx = code;
            asm volatile("{\n\tQGJ_TBL: .branchtargets " QGJ_LIST_6 ";\n\tbrx.idx %0, QGJ_TBL;\n\t}" ::"r"(idx));
        } else if constexpr (RB == 5) {
            static_assert(QGJ_N_5 == oc_xf(5), "jt_lists.h out of date");
            const uint32_t idx = code;
            asm volatile("{\n\tQGJ_TBL: .branchtargets " QGJ_LIST_5 ";\n\tbrx.idx %0, QGJ_TBL;\n\t}" ::"r"(idx));
        } else if constexpr (RB == 4) {
            static_assert(QGJ_N_4 == oc_xf(4), "jt_lists.h out of date");
            const uint32_t idx = code;
            asm volatile("{\n\tQGJ_TBL: .branchtargets " QGJ_LIST_4 ";\n\tbrx.idx %0, QGJ_TBL;\n\t}" ::"r"(idx));
        } else {
            static_assert(RB == 3, "jump tables exist for RB = 3, 4, 5, 6");
            static_assert(QGJ_N_3 == oc_xf(3), "jt_lists.h out of date");
            const uint32_t idx = code;
            asm volatile("{\n\tQGJ_TBL: .branchtargets " QGJ_LIST_3 ";\n\tbrx.idx %0, QGJ_TBL;\n\t}" ::"r"(idx));
        }
    }
#endif
    switch (w & 0xffu) {
#define QG_STD(T)                                                                        \
    case QG_LAB(T < RB, oc_std(F_RD, RB, T), T):                                         \
        if constexpr (T < RB) {                                                          \
            QGJ_ENTER("QGJ_RD_" #T);                                                     \
            op_rd<RB, 1u << T, 1u << T>(a, P.coef + (w >> 16), F);                       \
        }                                                                                \
        break;                                                                           \
    case QG_LAB(T < RB, oc_std(F_CD, RB, T), 8 + T):                                     \
        if constexpr (T < RB) {                                                          \
            QGJ_ENTER("QGJ_CD_" #T);                                                     \
            op_cd<RB, 1u << T, 1u << T>(a, P.coef + (w >> 16), F);                       \
        }                                                                                \
        break;                                                                           \
    case QG_LAB(T < RB, oc_std(F_PH, RB, T), 16 + T):                                    \
        if constexpr (T < RB) {                                                          \
            QGJ_ENTER("QGJ_PH_" #T);                                                     \
            op_ph<RB, 1u << T, T2, Real>(a, ph_product<UPH, T2>(P, w, tb), F);                \
        }                                                                                \
        break;
        QG_STD(0) QG_STD(1) QG_STD(2) QG_STD(3) QG_STD(4) QG_STD(5)
#undef QG_STD
#define QG_OKP(T, C) (T < RB && C < RB && T != C)
#define QG_PAIR(T, C)                                                                    \
    case QG_LAB(QG_OKP(T, C), oc_pair(F_RDW, RB, T, C), 100 + 6 * T + C):                \
        if constexpr (QG_OKP(T, C)) {                                                    \
            QGJ_ENTER("QGJ_RDW_" #T "_" #C);                                             \
            op_rd<RB, 1u << T, (1u << T) | (1u << C)>(a, P.coef + (w >> 16), F);         \
        }                                                                                \
        break;                                                                           \
    case QG_LAB(QG_OKP(T, C), oc_pair(F_RDV, RB, T, C), 200 + 6 * T + C):                \
        if constexpr (QG_OKP(T, C)) {                                                    \
            QGJ_ENTER("QGJ_RDV_" #T "_" #C);                                             \
            op_rd<RB, (1u << T) | (1u << C), 1u << T>(a, P.coef + (w >> 16), F);         \
        }                                                                                \
        break;                                                                           \
    case QG_LAB(QG_OKP(T, C) && C < T, oc_tri(F_PHW, RB, T, C), 500 + 6 * T + C):        \
        if constexpr (QG_OKP(T, C) && C < T) {                                           \
            QGJ_ENTER("QGJ_PHW_" #T "_" #C);                                             \
            op_ph<RB, (1u << T) | (1u << C), T2, Real>(a, ph_product<UPH, T2>(P, w, tb), F);  \
        }                                                                                \
        break;                                                                           \
    case QG_LAB(QG_OKP(T, C) && C < T, oc_tri(F_PH2, RB, T, C), 600 + 6 * T + C):        \
        if constexpr (QG_OKP(T, C) && C < T) {                                           \
            QGJ_ENTER("QGJ_PH2_" #T "_" #C);                                             \
            const Real* m = P.coef + (w >> 16);                                          \
            T2 e;                                                                        \
            e.x = m[0]; e.y = m[1];                                                      \
            const uint32_t ft = (F >> T) & 1u, fc = (F >> C) & 1u;                       \
            if (__ballot_sync(0xffffffffu, ft | fc) == 0u) r_cphase<RB, T, C>(a, e);     \
            else r_cphase_flip<RB, T, C>(a, e, ft, fc);                                  \
        }                                                                                \
        break;
#define QG_CXM(T, C)                                                                     \
    case QG_LAB(QG_OKP(T, C), oc_cxm(RB, T, C), 700 + 6 * T + C):                        \
        if constexpr (QG_OKP(T, C)) {                                                    \
            QGJ_ENTER("QGJ_CXM_" #T "_" #C);                                             \
            r_cx<RB, T, C>(a);                                                           \
            F ^= ((F >> C) & 1u) << T;                                                   \
        }                                                                                \
        break;
#define QG_CXMT(T) QG_CXM(T, 0) QG_CXM(T, 1) QG_CXM(T, 2) QG_CXM(T, 3) QG_CXM(T, 4) QG_CXM(T, 5)
        QG_CXMT(0) QG_CXMT(1) QG_CXMT(2) QG_CXMT(3) QG_CXMT(4) QG_CXMT(5)
#undef QG_CXMT
#undef QG_CXM
#define QG_PAIRT(T) QG_PAIR(T, 0) QG_PAIR(T, 1) QG_PAIR(T, 2) QG_PAIR(T, 3) QG_PAIR(T, 4) QG_PAIR(T, 5)
        QG_PAIRT(0) QG_PAIRT(1) QG_PAIRT(2) QG_PAIRT(3) QG_PAIRT(4) QG_PAIRT(5)
#undef QG_PAIRT
#undef QG_PAIR
#undef QG_OKP
        case oc_xf(RB): {
            QGJ_ENTER("QGJ_XF");
            const int n = (w >> 8) & 0xffu, b = w >> 16;
            for (int k = 0; k < n; ++k) {
                const uint32_t e = P.xfe[b + k];
                const uint32_t on = (uint32_t)(tb >> (e & 63u)) & 1u;
                F ^= (e >> 8) & (0u - on);
            }
            break;
        }
        case oc_end(RB): {
            QGJ_ENTER("QGJ_END");
            return;
        }
        default: __builtin_unreachable();
    }
    w = wn;
  }
}
#undef QG_LAB
#undef QGJ_ENTER

// ----------------------------------------------------------------- mappings
// SMEM offsets are kept in BYTES (swizzled amplitude index * sizeof(T2)) so an
// access is one LOP3 (xor) + STS/LDS [reg + smem_base] with no scaling.
template <int RB, typename T2>
__device__ __forceinline__ void smem_put(char* sm, const StageDesc& S, uint32_t so, const T2 (&a)[1 << RB],
                                         uint32_t F) {
    uint32_t rs[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) rs[b] = S.out_s[b];
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
    uint32_t rs[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) rs[b] = S.reg_s[b];
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
constexpr size_t kUphBytes = kMaxUph * 16;  // tile-uniform phase slots (T2 each), at offset 0
__host__ __device__ constexpr size_t tables_bytes() {  // + the tile-uniform phase slots
    return 4 * 256 * 8 + (kMaxStages + 1) * (kMapG * 8 + kMapS * 4) + kUphBytes;
}

// NBUF = 2: transposes alternate two tile buffers (one barrier each);
// NBUF = 1: one buffer, a second barrier before it is rewritten (half the SMEM,
// so two CTAs fit on an SM)
template <typename Real, int RB, int WB, int NBUF, bool UPH>
__global__ void __launch_bounds__(32 << WB, (WB >= 4 || sizeof(Real) == 8 || RB >= 6) ? 1 : 2)
    fused_pass_kernel(const __grid_constant__ PassDesc<Real> P, typename V2<Real>::T* __restrict__ psi,
                      uint64_t rank_bits) {
    using T2 = typename V2<Real>::T;
    constexpr int R = 1 << RB;
    constexpr int NT = 32 << WB;
    constexpr int sh = sizeof(T2) == 8 ? 3 : 4;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // [tile-uniform phase slots (UPH variant) | tile buffer(s) | index tables]; the
    // slots sit at a fixed address so the PH bodies need no pointer register
    char* sm = reinterpret_cast<char*>(smem_raw) + (UPH ? kUphBytes : 0);
    const int k = P.k;
    const uint32_t buf_bytes = (uint32_t)sizeof(T2) << k;
    uint64_t* tbase = reinterpret_cast<uint64_t*>(sm + NBUF * (size_t)buf_bytes);
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
        // the tile's amplitudes: pt[o], pt = psi + (the tile-id bits), o = the tile
        // bits; when every tile bit is below 32 (P.tile_lo32) the per-amplitude
        // address walk is 32-bit (1 LOP3 + 1 IMAD.WIDE instead of 64-bit XOR + LEA pair)
        T2* __restrict__ pt = psi + base;
        // opaque to the compiler, so psi + base + o is not re-associated into a
        // 64-bit add + LEA pair per amplitude: one IMAD.WIDE.U32 (o * 8 + pt) each
        asm("mov.b64 %0, %0;" : "+l"(pt));
        if (P.tile_lo32) {  // global load, Gray-code order over the register index
            const StageDesc& S = P.stg[li];
            uint32_t o = (uint32_t)tgb(li);
#pragma unroll
            for (int j = 0; j < R; ++j) {
                if (j) o ^= 1u << S.reg_q[ctz_c(j)];
                a[gray_c(j)] = __ldcs(pt + o);
            }
        } else {
            const StageDesc& S = P.stg[li];
            uint64_t g = tgb(li);
#pragma unroll
            for (int j = 0; j < R; ++j) {
                if (j) g ^= 1ull << S.reg_q[ctz_c(j)];
                a[gray_c(j)] = __ldcs(pt + g);
            }
        }
        {  // warm L2 with this CTA's next tile while this one computes: each of the
           // first R lanes prefetches one 32-amplitude run (2-4 lines, no registers held)
            const uint64_t nt = tile + gridDim.x;
            if (nt < P.n_tiles && lane < R) {
                const StageDesc& S = P.stg[li];
                uint64_t g = tbase[nt & 255] | tbase[256 + ((nt >> 8) & 255)] | tbase[512 + ((nt >> 16) & 255)] |
                             tbase[768 + ((nt >> 24) & 255)] | tmg[li * kMapG + 32 + warp];
#pragma unroll
                for (int b = 0; b < RB; ++b)
                    if ((lane >> b) & 1) g |= 1ull << S.reg_q[b];
                const char* p = reinterpret_cast<const char*>(psi + g);
#pragma unroll
                for (int l = 0; l < (int)(32 * sizeof(T2)) / 128; ++l)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(p + 128 * l));
            }
        }
        if constexpr (UPH) {  // tile-uniform phase slots (tile-id / rank bit factors): one warp
                              // per slot, its lanes splitting the factors, then a product tree
            const uint64_t ub = base | rank_bits;
            __syncthreads();  // every thread is done with the previous tile's slots
            for (int u = warp; u < P.n_uph; u += NT / 32) {
                const uint32_t d = P.uph[u];
                T2 e;
                e.x = Real(1);
                e.y = Real(0);
                for (uint32_t i = lane; i < (d >> 16); i += 32) {
                    const PhEnt<Real>& E = P.ph[(d & 0xffffu) + i];
                    if ((ub >> E.pos) & 1u) {
                        T2 v;
                        v.x = E.e[0];
                        v.y = E.e[1];
                        e = cmul(e, v);
                    }
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    T2 v;
                    v.x = __shfl_xor_sync(0xffffffffu, e.x, o);
                    v.y = __shfl_xor_sync(0xffffffffu, e.y, o);
                    e = cmul(e, v);
                }
                if (lane == 0) reinterpret_cast<T2*>(smem_raw)[u] = e;
            }
            __syncthreads();
        }
        int cur = li;
        uint32_t F = 0;  // register flip mask (see run_round)
        for (int s = 1; s <= ns; ++s) {
            const StageDesc& S = P.stg[s];
            if (cur != s) {  // SMEM transpose into this stage's mapping
                if (NBUF == 1) __syncthreads();  // every thread has read the previous transpose
                smem_put<RB>(sm + buf, P.stg[cur], tso(cur), a, F);
                __syncthreads();
                smem_get<RB>(sm + buf, S, tso(s), a);
                if (NBUF == 2) buf ^= buf_bytes;
                cur = s;
                F = 0;
            }
            const uint64_t tb = base | rank_bits | tgb(s);
            run_stage_ops<RB, UPH>(a, P, S.op_begin, tb, F);
            if (S.tph_end > S.tph_begin) {  // thread-level phases commute with the whole stage
                T2 ph;
                ph.x = Real(1);
                ph.y = Real(0);
                for (int e = S.tph_begin; e < S.tph_end; ++e) {
                    const Entry<Real>& E = P.tph[e];
                    if ((tb & E.cmask) != E.cmask) continue;
                    const bool hi = (tb & E.qmask) != 0;
                    T2 v;
                    v.x = hi ? E.v[2] : E.v[0];
                    v.y = hi ? E.v[3] : E.v[1];
                    ph = cmul(ph, v);
                }
                if (ph.y == Real(0)) {  // a real factor (a pass's rotation scale): the same values
#pragma unroll
                    for (int i = 0; i < R; ++i) {
                        a[i].x *= ph.x;
                        a[i].y *= ph.x;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < R; ++i) a[i] = cmul(a[i], ph);
                }
            }
        }
        if (cur != si) {
            if (NBUF == 1) __syncthreads();
            smem_put<RB>(sm + buf, P.stg[cur], tso(cur), a, F);
            __syncthreads();
            smem_get<RB>(sm + buf, P.stg[si], tso(si), a);
            if (NBUF == 2) buf ^= buf_bytes;
            F = 0;
        }
        if (P.tile_lo32) {  // global store through the output mapping (CX map + flips folded in)
            const StageDesc& S = P.stg[si];
            uint32_t og[RB];
#pragma unroll
            for (int b = 0; b < RB; ++b) og[b] = (uint32_t)S.out_g[b];
            uint32_t o = (uint32_t)tgb(si);
#pragma unroll
            for (int b = 0; b < RB; ++b)
                if ((F >> b) & 1u) o ^= og[b];
#pragma unroll
            for (int j = 0; j < R; ++j) {
                if (j) o ^= og[ctz_c(j)];
                __stcs(pt + o, a[gray_c(j)]);
            }
        } else {
            const StageDesc& S = P.stg[si];
            uint64_t og[RB];
#pragma unroll
            for (int b = 0; b < RB; ++b) og[b] = S.out_g[b];
            uint64_t g = tgb(si);
#pragma unroll
            for (int b = 0; b < RB; ++b)
                if ((F >> b) & 1u) g ^= og[b];
#pragma unroll
            for (int j = 0; j < R; ++j) {
                if (j) g ^= og[ctz_c(j)];
                __stcs(pt + g, a[gray_c(j)]);
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
template <typename Real, int RB, int WB, int NBUF, bool UPH>
static cudaError_t launch_fused_u(const PassDesc<Real>& P, void* psi, uint64_t rank_bits, cudaStream_t st) {
    constexpr int threads = 32 << WB;
    const int k = RB + kLaneBits + WB;
    const size_t smem = NBUF * ((size_t)1 << k) * sizeof(typename V2<Real>::T) + tables_bytes();
    auto kern = fused_pass_kernel<Real, RB, WB, NBUF, UPH>;
    // per instantiation AND per device (the SMEM attribute is a per-device setting):
    // resident CTAs per SM x SMs
    constexpr int kDevs = 64;
    static int max_blocks_dev[kDevs] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kDevs) return cudaErrorInvalidDevice;
    int& max_blocks = max_blocks_dev[dev];
    if (max_blocks <= 0) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int sms = 0, occ = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        if (e != cudaSuccess) return e;
        max_blocks = sms * (occ > 0 ? occ : 1);
    }
    const uint64_t grid = P.n_tiles < (uint64_t)max_blocks ? P.n_tiles : (uint64_t)max_blocks;
    kern<<<(unsigned)grid, threads, smem, st>>>(P, reinterpret_cast<typename V2<Real>::T*>(psi), rank_bits);
    return cudaGetLastError();
}

// passes without tile-uniform phase slots run the variant without their per-tile
// prologue and per-op flag test
template <typename Real, int RB, int WB, int NBUF = 2>
static cudaError_t launch_fused_t(const PassDesc<Real>& P, void* psi, uint64_t rank_bits, cudaStream_t st) {
    return P.n_uph ? launch_fused_u<Real, RB, WB, NBUF, true>(P, psi, rank_bits, st)
                   : launch_fused_u<Real, RB, WB, NBUF, false>(P, psi, rank_bits, st);
}

cudaError_t launch_fused(int dtype, int cfg_id, const void* desc, void* psi, uint64_t rank_bits, cudaStream_t st) {
    // must match kCfgC64 / kCfgC128 in plan.cpp
    if (dtype == 0) {
        const auto& P = *static_cast<const PassDesc<float>*>(desc);
        switch (cfg_id) {
            case 0: return launch_fused_t<float, 4, 4>(P, psi, rank_bits, st);
            case 1: return launch_fused_t<float, 4, 3>(P, psi, rank_bits, st);
            case 2: return launch_fused_t<float, 4, 2>(P, psi, rank_bits, st);
            case 4: return launch_fused_t<float, 5, 3, 1>(P, psi, rank_bits, st);
            case 5: return launch_fused_t<float, 5, 4, 1>(P, psi, rank_bits, st);
            case 6: return launch_fused_t<float, 5, 2, 1>(P, psi, rank_bits, st);
            case 7: return launch_fused_t<float, 6, 3, 1>(P, psi, rank_bits, st);
            case 8: return launch_fused_t<float, 6, 2, 1>(P, psi, rank_bits, st);
            default: return launch_fused_t<float, 3, 0>(P, psi, rank_bits, st);
        }
    }
    const auto& P = *static_cast<const PassDesc<double>*>(desc);
    switch (cfg_id) {
        case 0: return launch_fused_t<double, 4, 3>(P, psi, rank_bits, st);
        case 1: return launch_fused_t<double, 3, 2>(P, psi, rank_bits, st);
        case 3: return launch_fused_t<double, 5, 3, 1>(P, psi, rank_bits, st);
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
