// reduce.cu — state init, fp64 norm / probabilities, and the shot sampler.
//
// Reference: init_zero_state statevec.py:81-94; StateVector.norm_sq
// statevec.py:47-50; exact_probabilities statevec.py:215-218; sample_counts
// statevec.py:221-234 (fp64 |a|^2, norm check, cdf = cumsum / last,
// searchsorted(side='right') of uniforms, unique counts).
//
// Sampler (two-level inverse-CDF, no full-length prefix array):
//   1. chunk_sums:  one HBM read of the state; fp64 sums per 256-amp sub-block
//                   and per 16384-amp chunk (sub-block sums kept in workspace).
//   2. scan:        CUB exclusive prefix of the chunk sums (+ one 0) -> total.
//   3. draw:        per shot, u*total -> binary search over chunk prefixes ->
//                   linear walk over <= 64 sub-block sums -> <= 256 amplitudes.
//   4. (caller uniforms only) CUB radix sort of the outcomes; run-length encode
//      -> (index, count).
// Uniforms come from a counter-based Philox4x32-10 stream (seed, shot) turned into
// ascending order statistics (exponential spacings: no sort of the outcomes), or
// from the caller (numpy's default_rng(seed).random(shots) reproduces the
// reference's Generator.choice draws exactly up to fp64 rounding of the cdf;
// those outcomes are radix-sorted before the run-length encode).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cub/cub.cuh>
#include <cmath>

#include "kernels.h"

namespace qg {

template <typename Real>
struct A2;
template <>
struct A2<float> {
    using T = float2;
};
template <>
struct A2<double> {
    using T = double2;
};

template <typename T2>
__device__ __forceinline__ double prob(T2 a) {
    const double x = (double)a.x, y = (double)a.y;
    return x * x + y * y;
}

// ----------------------------------------------------------------- init
template <typename T2>
__global__ void set_one(T2* psi) {
    T2 v;
    v.x = 1;
    v.y = 0;
    psi[0] = v;
}

cudaError_t launch_init_zero(void* psi, int n_local, int dtype, int rank, cudaStream_t st) {
    const size_t bytes = ((size_t)1 << n_local) * (dtype == 0 ? 8 : 16);
    cudaError_t e = cudaMemsetAsync(psi, 0, bytes, st);
    if (e != cudaSuccess) return e;
    if (rank == 0) {
        if (dtype == 0) set_one<<<1, 1, 0, st>>>(static_cast<float2*>(psi));
        else set_one<<<1, 1, 0, st>>>(static_cast<double2*>(psi));
    }
    return cudaGetLastError();
}

// H on every qubit of `mask` applied to |0...0>: 2^(-|mask|/2) where the global
// index has no bit outside mask, 0 elsewhere (one write pass)
template <typename T2>
__global__ void set_uniform(T2* __restrict__ psi, uint64_t n, uint64_t rank_bits, uint64_t mask, double v) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        T2 a;
        a.x = ((rank_bits | i) & ~mask) ? 0 : v;
        a.y = 0;
        psi[i] = a;
    }
}

cudaError_t launch_init_uniform(void* psi, int n_local, int dtype, int rank, uint64_t mask, cudaStream_t st) {
    const uint64_t n = 1ull << n_local;
    const double v = std::pow(2.0, -0.5 * __builtin_popcountll(mask));
    const uint64_t rank_bits = (uint64_t)rank << n_local;
    const int threads = 256;
    uint64_t blocks = (n + threads - 1) / threads;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    if (dtype == 0) set_uniform<<<(unsigned)blocks, threads, 0, st>>>(static_cast<float2*>(psi), n, rank_bits, mask, v);
    else set_uniform<<<(unsigned)blocks, threads, 0, st>>>(static_cast<double2*>(psi), n, rank_bits, mask, v);
    return cudaGetLastError();
}

// ----------------------------------------------------------------- norm / probs
constexpr int kNormParts = 148 * 4;
int norm_parts() { return kNormParts; }

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    if (w == 0) {
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;  // valid in thread 0
}

template <typename T2>
__global__ void norm_partial(const T2* __restrict__ psi, int64_t n, double* __restrict__ part) {
    double acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += prob(psi[i]);
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void norm_finish(double* part, int n_parts) {
    double acc = 0;
    for (int i = threadIdx.x; i < n_parts; i += blockDim.x) acc += part[i];
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[n_parts] = acc;
}

cudaError_t launch_norm(const void* psi, int64_t n_amps, int dtype, double* partial, int n_parts, cudaStream_t st) {
    if (dtype == 0) norm_partial<<<n_parts, 256, 0, st>>>(static_cast<const float2*>(psi), n_amps, partial);
    else norm_partial<<<n_parts, 256, 0, st>>>(static_cast<const double2*>(psi), n_amps, partial);
    norm_finish<<<1, 1024, 0, st>>>(partial, n_parts);
    return cudaGetLastError();
}

template <typename T2>
__global__ void probs_kernel(const T2* __restrict__ psi, int64_t n, double* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = prob(psi[i]);
}

cudaError_t launch_probs(const void* psi, int64_t n_amps, int dtype, double* out, cudaStream_t st) {
    int64_t blocks = (n_amps + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (dtype == 0) probs_kernel<<<(int)blocks, 256, 0, st>>>(static_cast<const float2*>(psi), n_amps, out);
    else probs_kernel<<<(int)blocks, 256, 0, st>>>(static_cast<const double2*>(psi), n_amps, out);
    return cudaGetLastError();
}

// ----------------------------------------------------------------- sampler layout
constexpr int64_t kSub = 256;      // amplitudes per sub-block
constexpr int64_t kChunk = 16384;  // amplitudes per chunk (64 sub-blocks)

struct SLayout {
    int64_t sb, ch, n_sub, n_ch;
    size_t off_sub, off_bsum, off_bpre, off_draw, off_sorted, off_exp, off_runs, off_cub, total;
    size_t cub_bytes;
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static int bits_for(int64_t n) {
    int b = 0;
    while ((1ll << b) < n) ++b;
    return b < 1 ? 1 : b;
}

static SLayout layout(int64_t n_amps, int64_t shots) {
    SLayout L{};
    L.sb = n_amps < kSub ? n_amps : kSub;
    L.ch = n_amps < kChunk ? n_amps : kChunk;
    L.n_sub = n_amps / L.sb;
    L.n_ch = n_amps / L.ch;
    size_t sort_b = 0, rle_b = 0;
    const int64_t ns = shots > 0 ? shots : 1;
    cub::DeviceRadixSort::SortKeys(nullptr, sort_b, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                   (int)ns, 0, bits_for(n_amps));
    cub::DeviceRunLengthEncode::Encode(nullptr, rle_b, (const int64_t*)nullptr, (int64_t*)nullptr, (int64_t*)nullptr,
                                       (int64_t*)nullptr, (int)ns);
    size_t scan_b = 0;  // exclusive scan of the n_ch + 1 chunk sums (the last one 0 -> the total)
    cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (const double*)nullptr, (double*)nullptr, (int)(L.n_ch + 1));
    size_t cum_b = 0;  // inclusive scan of shots + 1 exponential spacings (sorted uniforms)
    cub::DeviceScan::InclusiveSum(nullptr, cum_b, (const double*)nullptr, (double*)nullptr, (int)(ns + 1));
    L.cub_bytes = std::max(std::max(sort_b, rle_b), std::max(scan_b, cum_b));
    size_t o = 0;
    L.off_sub = o; o += align256(L.n_sub * 8);
    L.off_bsum = o; o += align256((L.n_ch + 1) * 8);
    L.off_bpre = o; o += align256((L.n_ch + 1) * 8);
    L.off_draw = o; o += align256(ns * 8);
    L.off_sorted = o; o += align256((ns + 1) * 8);
    L.off_exp = o; o += align256((ns + 1) * 8);
    L.off_runs = o; o += align256(8);
    L.off_cub = o; o += align256(L.cub_bytes);
    L.total = o;
    return L;
}

int64_t sample_workspace_bytes(int64_t n_amps, int64_t shots) { return (int64_t)layout(n_amps, shots).total; }

const double* sample_total_ptr(const void* ws, int64_t n_amps) {
    const SLayout L = layout(n_amps, 1);
    return reinterpret_cast<const double*>(static_cast<const char*>(ws) + L.off_bpre) + L.n_ch;
}

const int64_t* sample_nunique_ptr(const void* ws, int64_t n_amps, int64_t shots) {
    const SLayout L = layout(n_amps, shots);
    return reinterpret_cast<const int64_t*>(static_cast<const char*>(ws) + L.off_runs);
}

// ----------------------------------------------------------------- sampler kernels
// 16-byte vector of amplitudes and its probability mass
template <typename T2>
struct Vec16;
template <>
struct Vec16<float2> {
    using T = float4;  // two complex64 amplitudes
    __device__ static double prob(float4 v) {
        const double a = v.x, b = v.y, c = v.z, d = v.w;
        return (a * a + b * b) + (c * c + d * d);
    }
};
template <>
struct Vec16<double2> {
    using T = double2;  // one complex128 amplitude
    __device__ static double prob(double2 v) { return v.x * v.x + v.y * v.y; }
};

// one CTA (256 threads = 8 warps) per chunk; warp w sums sub-blocks w, w+8, ...
template <typename T2>
__global__ void chunk_sums(const T2* __restrict__ psi, int64_t sb, int64_t ch, double* __restrict__ sub,
                           double* __restrict__ bsum) {
    const int64_t c = blockIdx.x;
    const int64_t nsb = ch / sb;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    double wacc = 0;
    for (int64_t j = w; j < nsb; j += 8) {
        const T2* p = psi + c * ch + j * sb;
        double acc = 0;
        if (sb == kSub) {
            // lane l owns amplitudes [8l, 8l + 8) of the sub-block: every 16-byte
            // load is issued before the first use (the scalar loop kept one in flight)
            using V = typename Vec16<T2>::T;
            constexpr int kA = 16 / (int)sizeof(T2);  // amplitudes per vector
            const V* pv = reinterpret_cast<const V*>(p) + l * (8 / kA);
            V v[8 / kA];
#pragma unroll
            for (int k = 0; k < 8 / kA; ++k) v[k] = __ldcs(pv + k);
#pragma unroll
            for (int k = 0; k < 8 / kA; ++k) acc += Vec16<T2>::prob(v[k]);
        } else {
            for (int64_t i = l; i < sb; i += 32) acc += prob(p[i]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (l == 0) sub[c * nsb + j] = acc;
        wacc += acc;
    }
    __shared__ double ws[8];
    if (l == 0) ws[w] = wacc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int i = 0; i < 8; ++i) t += ws[i];
        bsum[c] = t;
        if (c == 0) bsum[gridDim.x] = 0.0;  // the scan's extra element
    }
}

__device__ __forceinline__ uint32_t mulhilo(uint32_t a, uint32_t b, uint32_t& hi) {
    const uint64_t p = (uint64_t)a * b;
    hi = (uint32_t)(p >> 32);
    return (uint32_t)p;
}

// Philox4x32-10 (Salmon et al., SC'11) -> one double in [0, 1) with 53 random bits
__device__ __forceinline__ double philox_uniform(uint64_t seed, uint64_t ctr) {
    uint32_t c0 = (uint32_t)ctr, c1 = (uint32_t)(ctr >> 32), c2 = 0x51ea1e5u, c3 = 0u;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, hi1;
        const uint32_t lo0 = mulhilo(0xD2511F53u, c0, hi0);
        const uint32_t lo1 = mulhilo(0xCD9E8D57u, c2, hi1);
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    const uint64_t x = ((uint64_t)c0 << 32) | c1;
    return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

// Exp(1) variates from the Philox stream: their running sums S_1..S_{N+1} give the
// order statistics of N uniforms as S_k / S_{N+1} (exactly distributed as sorted
// uniforms), so the draws come out in index order and need no sort
__global__ void expo_kernel(uint64_t seed, int64_t m, double* __restrict__ out) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < m; s += (int64_t)gridDim.x * blockDim.x)
        out[s] = -log1p(-philox_uniform(seed, (uint64_t)s));
}

// uni = caller uniforms (any order), or the running exponential sums with their
// total at uni_total (ascending uniforms); out[s] = the outcome of draw s
template <typename T2>
__global__ void draw_kernel(const T2* __restrict__ psi, int64_t shots, const double* __restrict__ uni,
                            const double* __restrict__ uni_total, const double* __restrict__ sub,
                            const double* __restrict__ bpre, int64_t n_ch, int64_t sb, int64_t ch,
                            unsigned long long* __restrict__ out) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= shots) return;
    const double u = uni_total ? uni[s] / *uni_total : uni[s];
    const double tot = bpre[n_ch];
    const double target = u * tot;
    // first chunk c with bpre[c+1] > target  (searchsorted side='right')
    int64_t lo = 0, hi = n_ch - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (bpre[mid + 1] > target) hi = mid;
        else lo = mid + 1;
    }
    int64_t c = lo;
    while (c > 0 && bpre[c + 1] - bpre[c] <= 0.0) --c;  // rounding clamp onto a chunk with mass
    double r = target - bpre[c];
    // two sequential scans (sub-block sums, then the sub-block's amplitudes), each
    // reading kB values per batch with independent loads; the compare / accumulate
    // order is the plain left-to-right loop's, so the outcome is bit-for-bit the same
    constexpr int kB = 16;
    const int64_t nsb = ch / sb;
    int64_t j = nsb, last = -1;
    double acc = 0;
    for (int64_t j0 = 0; j0 < nsb && j == nsb; j0 += kB) {
        double v[kB];
#pragma unroll
        for (int k = 0; k < kB; ++k) v[k] = j0 + k < nsb ? sub[c * nsb + j0 + k] : 0.0;
#pragma unroll
        for (int k = 0; k < kB; ++k) {
            if (j0 + k >= nsb) break;
            if (v[k] > 0) last = j0 + k;
            if (acc + v[k] > r) { j = j0 + k; break; }
            acc += v[k];
        }
    }
    if (j == nsb) { j = last < 0 ? nsb - 1 : last; acc -= sub[c * nsb + j]; }
    r -= acc;
    const T2* p = psi + c * ch + j * sb;
    int64_t i = sb, lasti = -1;
    double acc2 = 0;
    for (int64_t i0 = 0; i0 < sb && i == sb; i0 += kB) {
        double v[kB];
#pragma unroll
        for (int k = 0; k < kB; ++k) v[k] = i0 + k < sb ? prob(p[i0 + k]) : 0.0;
#pragma unroll
        for (int k = 0; k < kB; ++k) {
            if (i0 + k >= sb) break;
            if (v[k] > 0) lasti = i0 + k;
            if (acc2 + v[k] > r) { i = i0 + k; break; }
            acc2 += v[k];
        }
    }
    if (i == sb) i = lasti < 0 ? sb - 1 : lasti;
    out[s] = (unsigned long long)(c * ch + j * sb + i);
}

cudaError_t sample_prefix(const void* psi, int64_t n_amps, int dtype, void* ws, cudaStream_t st, double* total_dev) {
    const SLayout L = layout(n_amps, 1);
    char* w = static_cast<char*>(ws);
    double* sub = reinterpret_cast<double*>(w + L.off_sub);
    double* bsum = reinterpret_cast<double*>(w + L.off_bsum);
    double* bpre = reinterpret_cast<double*>(w + L.off_bpre);
    if (dtype == 0) chunk_sums<<<(unsigned)L.n_ch, 256, 0, st>>>(static_cast<const float2*>(psi), L.sb, L.ch, sub, bsum);
    else chunk_sums<<<(unsigned)L.n_ch, 256, 0, st>>>(static_cast<const double2*>(psi), L.sb, L.ch, sub, bsum);
    size_t tb = L.cub_bytes;  // bsum[n_ch] = 0 (chunk_sums), so bpre[n_ch] = the total
    cudaError_t e = cub::DeviceScan::ExclusiveSum(w + L.off_cub, tb, bsum, bpre, (int)(L.n_ch + 1), st);
    if (e != cudaSuccess) return e;
    (void)total_dev;
    return cudaGetLastError();
}

cudaError_t sample_draw(const void* psi, int64_t n_amps, int dtype, int64_t shots, uint64_t seed,
                        const double* uniforms, void* ws, int64_t* out_idx, int64_t* out_cnt, cudaStream_t st,
                        int64_t* n_unique_dev) {
    const SLayout L = layout(n_amps, shots);
    char* w = static_cast<char*>(ws);
    const double* sub = reinterpret_cast<const double*>(w + L.off_sub);
    const double* bpre = reinterpret_cast<const double*>(w + L.off_bpre);
    auto* draws = reinterpret_cast<unsigned long long*>(w + L.off_draw);
    auto* sorted = reinterpret_cast<unsigned long long*>(w + L.off_sorted);
    const unsigned blocks = (unsigned)((shots + 63) / 64);  // latency-bound threads: spread over SMs
    const double* uni = uniforms;
    const double* uni_total = nullptr;
    cudaError_t e;
    size_t tb = L.cub_bytes;
    if (!uniforms) {  // Philox stream as ascending uniforms (exponential spacings)
        double* ex = reinterpret_cast<double*>(w + L.off_exp);
        double* cum = reinterpret_cast<double*>(w + L.off_sorted);
        const int64_t m = shots + 1;
        const unsigned eb = (unsigned)std::min<int64_t>((m + 255) / 256, 148 * 16);
        expo_kernel<<<eb, 256, 0, st>>>(seed, m, ex);
        e = cub::DeviceScan::InclusiveSum(w + L.off_cub, tb, ex, cum, (int)m, st);
        if (e != cudaSuccess) return e;
        uni = cum;
        uni_total = cum + shots;
    }
    if (dtype == 0)
        draw_kernel<<<blocks, 64, 0, st>>>(static_cast<const float2*>(psi), shots, uni, uni_total, sub, bpre, L.n_ch,
                                            L.sb, L.ch, draws);
    else
        draw_kernel<<<blocks, 64, 0, st>>>(static_cast<const double2*>(psi), shots, uni, uni_total, sub, bpre,
                                            L.n_ch, L.sb, L.ch, draws);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const unsigned long long* keys = draws;  // ascending already for the Philox stream
    if (uniforms) {
        tb = L.cub_bytes;
        e = cub::DeviceRadixSort::SortKeys(w + L.off_cub, tb, draws, sorted, (int)shots, 0, bits_for(n_amps), st);
        if (e != cudaSuccess) return e;
        keys = sorted;
    }
    tb = L.cub_bytes;
    e = cub::DeviceRunLengthEncode::Encode(w + L.off_cub, tb, reinterpret_cast<const int64_t*>(keys), out_idx,
                                           out_cnt, n_unique_dev, (int)shots, st);
    return e;
}

}  // namespace qg
