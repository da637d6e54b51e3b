// ucry.cu — uniformly controlled RY in one pass (QCrank's data-register rotation).
//
// QCrank writes each data qubit d with a uniformly controlled
// RY over the m address qubits: for address a the data qubit sees RY(alpha[a][d]).
// As gates this is the Gray-code block of 2^m RY + 2^m CX per data qubit
// (built by qcrank.build_qcrank_circuit) — 2.7e8 gates for the
// 24 + 8 qubit configuration, far beyond any gate-level planner.  The host
// recognises the block (qcrank.collapse_ucry: the Walsh-Hadamard transform in
// Gray order recovers alpha) and runs it here as one HBM pass for up to
// kMaxUcryTargets data qubits at once:
//
//   thread = one address a: it reads its cos/sin for every target once (a
//   per-address table built in fp64 and cast, like statevec.py:117), then for
//   each combination of the remaining qubits holds the 2^T amplitudes of its
//   T target qubits in registers, applies RY(alpha[a][d]) for every target d,
//   and writes them back.
//
// Traffic = read + write of the state once (+ the table, 2^m * T * 2 reals).
#include <cuda_runtime.h>

#include <algorithm>
#include <stdint.h>

#include "kernels.h"

namespace qg {

namespace {

template <typename Real>
struct U2;
template <>
struct U2<float> {
    using T = float2;
};
template <>
struct U2<double> {
    using T = double2;
};

// table[t][a] = (cos(alpha/2), sin(alpha/2)) in the state's precision, from fp64 angles
template <typename Real>
__global__ void ucry_table(const double* __restrict__ alpha, int64_t n_addr, int n_t,
                           typename U2<Real>::T* __restrict__ table) {
    const int64_t total = n_addr * n_t;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = e / n_t;
        const int t = (int)(e % n_t);
        double s, c;
        sincos(alpha[e] * 0.5, &s, &c);  // alpha is [a][t] row-major
        typename U2<Real>::T v;
        v.x = (Real)c;
        v.y = (Real)s;
        table[(int64_t)t * n_addr + a] = v;
    }
}

__device__ __forceinline__ uint64_t deposit(uint64_t v, const uint8_t* pos, int n) {
    uint64_t r = 0;
    for (int k = 0; k < n; ++k) r |= ((v >> k) & 1ull) << pos[k];
    return r;
}

template <typename Real, int T>
__global__ void __launch_bounds__(256) ucry_kernel(typename U2<Real>::T* __restrict__ psi, UcryOp op,
                                                   const typename U2<Real>::T* __restrict__ table) {
    using C2 = typename U2<Real>::T;
    const uint64_t n_addr = 1ull << op.m;
    const uint64_t n_rest = 1ull << op.n_rest;
    // thread = one address a: its cos/sin for every target are read once and
    // reused for all 2^n_rest combinations of the remaining qubits
    for (uint64_t a = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < n_addr;
         a += (uint64_t)gridDim.x * blockDim.x) {
        Real c[T], s[T];
#pragma unroll
        for (int k = 0; k < T; ++k) {
            const C2 cs = table[(uint64_t)k * n_addr + a];
            c[k] = cs.x;
            s[k] = cs.y;
        }
        const uint64_t abits = op.addr_contig ? (a << op.addr_pos[0]) : deposit(a, op.addr_pos, op.m);
        for (uint64_t r = 0; r < n_rest; ++r) {
            const uint64_t base = abits | deposit(r, op.rest_pos, op.n_rest);
            C2 v[1 << T];
#pragma unroll
            for (int x = 0; x < (1 << T); ++x) {
                uint64_t i = base;
#pragma unroll
                for (int k = 0; k < T; ++k) i |= (uint64_t)((x >> k) & 1) << op.tgt_pos[k];
                v[x] = psi[i];
            }
#pragma unroll
            for (int k = 0; k < T; ++k) {
#pragma unroll
                for (int x = 0; x < (1 << T); ++x) {
                    if (x & (1 << k)) continue;
                    const C2 p = v[x], q = v[x | (1 << k)];
                    C2 u, w;  // RY = [[c, -s], [s, c]] (statevec.py:104)
                    u.x = c[k] * p.x - s[k] * q.x;
                    u.y = c[k] * p.y - s[k] * q.y;
                    w.x = s[k] * p.x + c[k] * q.x;
                    w.y = s[k] * p.y + c[k] * q.y;
                    v[x] = u;
                    v[x | (1 << k)] = w;
                }
            }
#pragma unroll
            for (int x = 0; x < (1 << T); ++x) {
                uint64_t i = base;
#pragma unroll
                for (int k = 0; k < T; ++k) i |= (uint64_t)((x >> k) & 1) << op.tgt_pos[k];
                psi[i] = v[x];
            }
        }
    }
}

template <typename Real>
cudaError_t launch_t(void* psi, const UcryOp& op, const double* alpha, void* ws, cudaStream_t st) {
    using C2 = typename U2<Real>::T;
    C2* table = static_cast<C2*>(ws);
    const int64_t n_addr = 1ll << op.m;
    {
        const int64_t total = n_addr * op.n_t;
        const int threads = 256;
        int64_t blocks = (total + threads - 1) / threads;
        if (blocks > 148 * 32) blocks = 148 * 32;
        ucry_table<Real><<<(unsigned)blocks, threads, 0, st>>>(alpha, n_addr, op.n_t, table);
    }
    uint64_t blocks = ((uint64_t)n_addr + 255) / 256;
    if (blocks > 148ull * 8) blocks = 148ull * 8;
    C2* s = static_cast<C2*>(psi);
    switch (op.n_t) {
        case 1: ucry_kernel<Real, 1><<<(unsigned)blocks, 256, 0, st>>>(s, op, table); break;
        case 2: ucry_kernel<Real, 2><<<(unsigned)blocks, 256, 0, st>>>(s, op, table); break;
        case 3: ucry_kernel<Real, 3><<<(unsigned)blocks, 256, 0, st>>>(s, op, table); break;
        case 4: ucry_kernel<Real, 4><<<(unsigned)blocks, 256, 0, st>>>(s, op, table); break;
        default: ucry_kernel<Real, 5><<<(unsigned)blocks, 256, 0, st>>>(s, op, table); break;
    }
    return cudaGetLastError();
}

}  // namespace

int64_t ucry_workspace_bytes(int m, int n_t, int dtype) {
    return ((int64_t)1 << m) * n_t * (dtype == 0 ? 8 : 16);
}

cudaError_t launch_ucry(int dtype, void* psi, const UcryOp& op, const double* alpha_dev, void* ws, cudaStream_t st) {
    return dtype == 0 ? launch_t<float>(psi, op, alpha_dev, ws, st) : launch_t<double>(psi, op, alpha_dev, ws, st);
}

// QCrank decode tallies from dense per-outcome counts: outcome
// index = address (low m bits) + 2^m * data bits.  One thread per address walks its
// 2^n_data outcomes (a warp reads 32 consecutive addresses per outcome: coalesced):
// tot[a] = all shots at address a, n1[a * n_data + j] = those with data bit j = 1.
__global__ void qcrank_tally(const int64_t* __restrict__ dense, int m, int nd, int64_t* __restrict__ tot,
                             int64_t* __restrict__ n1) {
    const int64_t na = 1ll << m;
    for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < na; a += (int64_t)gridDim.x * blockDim.x) {
        int64_t t = 0, b[16] = {};
        for (int64_t d = 0; d < (1ll << nd); ++d) {
            const int64_t c = __ldcs(dense + a + (d << m));
            t += c;
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j < nd && ((d >> j) & 1)) b[j] += c;
        }
        tot[a] = t;
        for (int j = 0; j < nd; ++j) n1[a * nd + j] = b[j];
    }
}

cudaError_t launch_qcrank_tally(const int64_t* dense, int m, int nd, int64_t* tot, int64_t* n1, cudaStream_t st) {
    const int64_t na = 1ll << m;
    qcrank_tally<<<(unsigned)std::min<int64_t>((na + 255) / 256, 148 * 16), 256, 0, st>>>(dense, m, nd, tot, n1);
    return cudaGetLastError();
}

}  // namespace qg
