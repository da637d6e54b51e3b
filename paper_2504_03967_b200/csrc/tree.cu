// tree.cu — multinomial shot sampler by binomial splitting ("tree sampler").
//
// Reference: sample_counts (statevec.py:221-234) draws `shots` outcomes from
// p_i = |a_i|^2 / sum|a|^2 and tallies them.  The counts of a multinomial draw
// are generated here directly, top-down over the binary tree of the index bits:
// a node holding n shots with children masses (mL, mR) sends
// k ~ Binomial(n, mL / (mL + mR)) to the left child and n - k to the right.
// The result has exactly the multinomial distribution of `shots` independent
// draws (the conditional distributions of a multinomial are binomial), so it
// is a drop-in for the reference's Generator.choice + np.unique up to the
// random stream.  What this buys over per-shot inverse-CDF sampling:
//   * shots are int64 and never materialised: work and workspace are
//     O(amplitudes / 256), not O(shots) (QCrank: s * 2^m = 3000 * 2^24 ~ 5e10
//     shots);
//   * a sharded state samples without gathering it: the rank masses split the
//     shots first (qg_split_shots), then each rank runs its own subtree;
//   * the result is independent of the launch geometry: the split at tree node
//     (depth d, index i) draws from the Philox4x32-10 stream keyed by (seed) at
//     counter (i, d | tag << 8, j), j = 0, 1, ... for its rejection loop.
//
// Layout: leaves of the stored tree are 256-amplitude sub-blocks (one warp
// each); the mass and count trees over the n_sub sub-blocks are heap-ordered
// arrays (node (d, i) at (1 << d) - 1 + i).  Inside a sub-block the splits run
// across lane groups (shuffles) and then inside a lane (8 amplitudes).
// Binomial draws: BTRS (Hörmann 1993, transformed rejection with squeeze) for
// n·min(p, 1-p) >= 10, else the geometric waiting-time method — both exact.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cub/cub.cuh>
#include <type_traits>

#include "kernels.h"

namespace qg {

namespace {

constexpr int kSubT = 256;  // amplitudes per stored leaf (one warp, 8 per lane)

__device__ __forceinline__ uint4 philox4(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t key) {
    uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return make_uint4(c0, c1, c2, c3);
}

// uniforms in (0, 1) (never 0 or 1) for one tree node
struct NodeRng {
    uint64_t key;
    uint32_t c0, c1, c2, j = 0;
    int have = 0;
    double spare = 0;
    __device__ NodeRng(uint64_t seed, uint32_t tag, int depth, uint64_t idx)
        : key(seed), c0((uint32_t)idx), c1((uint32_t)(idx >> 32)), c2((uint32_t)depth | (tag << 8)) {}
    __device__ __forceinline__ double uni() {
        if (have) {
            have = 0;
            return spare;
        }
        const uint4 x = philox4(c0, c1, c2, j++, key);
        const uint64_t a = ((uint64_t)x.x << 32) | x.y, b = ((uint64_t)x.z << 32) | x.w;
        constexpr double s = 1.0 / 9007199254740992.0;  // 2^-53
        spare = ((double)(b >> 11) + 0.5) * s;
        have = 1;
        return ((double)(a >> 11) + 0.5) * s;
    }
};

// log(k!) - [(k + 1/2) log(k + 1) - (k + 1) + log(2 pi) / 2]  (Stirling series tail)
__constant__ double kStirlingTail[10] = {0.08106146679532733, 0.04134069595540946, 0.027677925684997717,
                                         0.02079067210376584, 0.01664469118982126, 0.013876128823072875,
                                         0.011896709945893313, 0.010411265261973668, 0.00925546218270945,
                                         0.008330563433359472};
__device__ __forceinline__ double stirling_tail(double k) {
    if (k <= 9) return kStirlingTail[(int)k];
    const double kp1sq = (k + 1) * (k + 1);
    return (1.0 / 12 - (1.0 / 360 - 1.0 / 1260 / kp1sq) / kp1sq) / (k + 1);
}

// Binomial(n, p), n a non-negative integer held exactly in a double (< 2^53)
__device__ double binomial(double n, double p, NodeRng& g) {
    if (n <= 0 || !(p > 0)) return 0;
    if (p >= 1) return n;
    const bool flip = p > 0.5;
    if (flip) p = 1 - p;
    double k;
    if (n * p < 10) {  // waiting time: count geometric(p) trial runs that fit in n trials
        const double logq = log1p(-p);
        double sum = 0;
        k = 0;
        for (;;) {
            sum += ceil(log(g.uni()) / logq);
            if (sum > n) break;
            k += 1;
        }
    } else {  // BTRS
        const double sd = sqrt(n * p * (1 - p));
        const double b = 1.15 + 2.53 * sd;
        const double a = -0.0873 + 0.0248 * b + 0.01 * p;
        const double c = n * p + 0.5;
        const double vr = 0.92 - 4.2 / b;
        const double r = p / (1 - p);
        const double alpha = (2.83 + 5.1 / b) * sd;
        const double m = floor((n + 1) * p);
        for (;;) {
            const double u = g.uni() - 0.5;
            double v = g.uni();
            const double us = 0.5 - fabs(u);
            k = floor((2 * a / us + b) * u + c);
            if (us >= 0.07 && v <= vr) break;
            if (k < 0 || k > n) continue;
            v = log(v * alpha / (a / (us * us) + b));
            const double ub = (m + 0.5) * log((m + 1) / (r * (n - m + 1))) + (n + 1) * log((n - m + 1) / (n - k + 1)) +
                              (k + 0.5) * log(r * (n - k + 1) / (k + 1)) + stirling_tail(m) + stirling_tail(n - m) -
                              stirling_tail(k) - stirling_tail(n - k);
            if (v <= ub) break;
        }
    }
    return flip ? n - k : k;
}

__device__ __forceinline__ double split(double n, double mL, double mR, uint64_t seed, uint32_t tag, int depth,
                                        uint64_t idx) {
    if (n <= 0) return 0;
    if (!(mR > 0)) return mL > 0 ? n : 0;  // all to the left (a zero-mass pair keeps nothing)
    if (!(mL > 0)) return 0;
    NodeRng g(seed, tag, depth, idx);
    return binomial(n, mL / (mL + mR), g);
}

template <typename T2>
__device__ __forceinline__ double pr(T2 a) {
    const double x = (double)a.x, y = (double)a.y;
    return x * x + y * y;
}

// per-lane amplitudes of a sub-block: lane l owns [l*A, l*A + A) (A = sb / 32, or 1 lane per amplitude)
template <typename T2>
__device__ __forceinline__ void lane_probs(const T2* __restrict__ p, int sb, int lane, double (&q)[8], int& A) {
    A = sb >= 32 ? sb / 32 : 1;
#pragma unroll
    for (int a = 0; a < 8; ++a) q[a] = 0;
    if (sb >= 256) {
#pragma unroll
        for (int a = 0; a < 8; ++a) q[a] = pr(__ldcs(p + lane * 8 + a));
    } else if (sb >= 32) {
        for (int a = 0; a < A; ++a) q[a] = pr(p[lane * A + a]);
    } else if (lane < sb) {
        q[0] = pr(p[lane]);
    }
}

// ---------------------------------------------------------------- up: masses
template <typename T2>
__global__ void leaf_mass(const T2* __restrict__ psi, int64_t n_sub, int sb, double* __restrict__ leaf) {
    const int lane = threadIdx.x & 31;
    const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (j >= n_sub) return;
    double q[8];
    int A;
    lane_probs(psi + j * sb, sb, lane, q, A);
    double m = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
    if (lane == 0) leaf[j] = m;
}

__global__ void tree_up(double* __restrict__ mass, int d) {  // level d from level d + 1
    const int64_t n = 1ll << d;
    double* up = mass + (n - 1);
    const double* dn = mass + (2 * n - 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        up[i] = dn[2 * i] + dn[2 * i + 1];
}

// ---------------------------------------------------------------- down: counts
__global__ void set_root(int64_t* cnt, int64_t shots) { cnt[0] = shots; }

__global__ void tree_down(const double* __restrict__ mass, int64_t* __restrict__ cnt, int d, uint64_t seed,
                          uint32_t tag) {
    const int64_t n = 1ll << d;
    const int64_t* c = cnt + (n - 1);
    int64_t* cd = cnt + (2 * n - 1);
    const double* md = mass + (2 * n - 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = c[i];
        const int64_t l = (int64_t)split((double)k, md[2 * i], md[2 * i + 1], seed, tag, d, (uint64_t)i);
        cd[2 * i] = l;
        cd[2 * i + 1] = k - l;
    }
}

// ---------------------------------------------------------------- leaves
// mode 0: nz[j] = outcomes with a count in sub-block j; mode 1: write (index, count)
// at nzpre[j]...; mode 2: dense counts (every amplitude, zeros included)
template <typename T2, int MODE>
__global__ void tree_leaf(const T2* __restrict__ psi, int64_t n_sub, int sb, int D, const int64_t* __restrict__ leaf_cnt,
                          uint64_t seed, uint32_t tag, int64_t idx_base, int64_t* __restrict__ nz,
                          const int64_t* __restrict__ nzpre, int64_t* __restrict__ out_idx,
                          int64_t* __restrict__ out_cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (j >= n_sub) return;
    const int64_t n0 = leaf_cnt[j];
    if (n0 == 0) {
        if (MODE == 0 && lane == 0) nz[j] = 0;
        if (MODE == 2)
            for (int a = lane; a < sb; a += 32) out_cnt[j * sb + a] = 0;
        return;
    }
    double q[8];
    int A;
    lane_probs(psi + j * sb, sb, lane, q, A);
    // lane-group masses: s[t] = sum over the aligned group of 2^t lanes
    double s[6];
    s[0] = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
#pragma unroll
    for (int t = 1; t < 6; ++t) s[t] = s[t - 1] + __shfl_xor_sync(0xffffffffu, s[t - 1], 1 << (t - 1));
    // lanes: depth D + t splits groups of 32 >> t lanes into halves (t = 0..4)
    double n = (double)n0;
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        const int G = 32 >> t, H = G >> 1;
        const int h = 4 - t;  // s index of the half-group
        const double mine = s[h], other = __shfl_xor_sync(0xffffffffu, s[h], H);
        const bool right = (lane & H) != 0;
        const double mL = right ? other : mine, mR = right ? mine : other;
        double k = 0;
        if ((lane & (G - 1)) == 0)
            k = split(n, mL, mR, seed, tag, D + t, ((uint64_t)j << t) + (uint64_t)(lane / G));
        k = __shfl_sync(0xffffffffu, k, lane & ~(G - 1));
        n = right ? n - k : k;
    }
    // inside the lane: depth D + 5 .. D + 7 over 8 amplitude slots
    double c[8];
    {
        const uint64_t node = ((uint64_t)j << 5) + (uint64_t)lane;  // depth D + 5
        const double l4 = (q[0] + q[1]) + (q[2] + q[3]), r4 = (q[4] + q[5]) + (q[6] + q[7]);
        const double k4 = split(n, l4, r4, seed, tag, D + 5, node);
        const double h[2] = {k4, n - k4};
        double g2[4];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const double l2 = q[4 * u] + q[4 * u + 1], r2 = q[4 * u + 2] + q[4 * u + 3];
            const double k2 = split(h[u], l2, r2, seed, tag, D + 6, node * 2 + u);
            g2[2 * u] = k2;
            g2[2 * u + 1] = h[u] - k2;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double k1 = split(g2[u], q[2 * u], q[2 * u + 1], seed, tag, D + 7, node * 4 + u);
            c[2 * u] = k1;
            c[2 * u + 1] = g2[u] - k1;
        }
    }
    // slot a of this lane is amplitude lane * A + a when a < A (A < 8 only for sb < 256:
    // the unused slots have zero mass and receive nothing)
    const int64_t base = j * sb;
    if (MODE == 2) {
        for (int a = 0; a < A; ++a)
            if (lane * A + a < sb) out_cnt[base + lane * A + a] = (int64_t)c[a];
        return;
    }
    int mine = 0;
#pragma unroll
    for (int a = 0; a < 8; ++a) mine += c[a] > 0 ? 1 : 0;
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (MODE == 0) {
        if (lane == 31) nz[j] = incl;
        return;
    }
    int64_t pos = nzpre[j] + (incl - mine);
    for (int a = 0; a < 8; ++a)
        if (c[a] > 0) {
            const int64_t amp = (sb >= 32) ? (int64_t)lane * A + a : (int64_t)lane;
            out_idx[pos] = idx_base + base + amp;
            out_cnt[pos] = (int64_t)c[a];
            ++pos;
        }
}

// ---------------------------------------------------------------- dense mode: level-synchronous
// Below the stored leaves the dense count array itself holds the tree: node (d, i)
// lives at position i << (nl - d), its left child at the same position, its right
// child at + half.  One level per launch, one binomial per node (a warp per node for
// ranges >= 64 amplitudes, a thread per node below): no dependency chains inside a
// warp, so the binomials run at the generator's throughput.  Children masses are
// balanced pairwise sums in index order — bitwise the sums tree_leaf forms with its
// in-lane adds and xor-butterflies — so both modes draw the same counts.
__global__ void scatter_leaves(const int64_t* __restrict__ leaf_cnt, int64_t n_sub, int sb_log,
                               int64_t* __restrict__ dense) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_sub; j += (int64_t)gridDim.x * blockDim.x)
        dense[j << sb_log] = leaf_cnt[j];
}

template <typename T2, int C>
__device__ __forceinline__ double tree_sum(const T2* __restrict__ p) {  // balanced pairwise sum of C amplitudes
    double v[C];
#pragma unroll
    for (int a = 0; a < C; ++a) v[a] = pr(p[a]);
#pragma unroll
    for (int w = 1; w < C; w <<= 1)
#pragma unroll
        for (int a = 0; a < C; a += 2 * w) v[a] += v[a + w];
    return v[0];
}

template <typename T2, int H>  // thread per node, children of H amplitudes (H <= 16)
__global__ void level_thread(const T2* __restrict__ psi, int64_t* __restrict__ dense, int nl, int d, uint64_t seed,
                             uint32_t tag) {
    const int64_t nn = 1ll << d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pos = i << (nl - d);
        const int64_t n = dense[pos];
        if (n == 0) {
            dense[pos + H] = 0;
            continue;
        }
        const double mL = tree_sum<T2, H>(psi + pos), mR = tree_sum<T2, H>(psi + pos + H);
        const int64_t k = (int64_t)split((double)n, mL, mR, seed, tag, d, (uint64_t)i);
        dense[pos] = k;
        dense[pos + H] = n - k;
    }
}

template <typename T2, int C>  // warp per node, each lane sums C consecutive amplitudes (node = 32 C amps)
__global__ void level_warp(const T2* __restrict__ psi, int64_t* __restrict__ dense, int nl, int d, uint64_t seed,
                           uint32_t tag) {
    const int lane = threadIdx.x & 31;
    const int64_t nn = 1ll << d;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int R = 32 * C;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nn; i += warps) {
        const int64_t pos = i * R;
        const int64_t n = dense[pos];
        if (n == 0) {
            if (lane == 0) dense[pos + R / 2] = 0;
            continue;
        }
        double m = tree_sum<T2, C>(psi + pos + (int64_t)lane * C);
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) m += __shfl_xor_sync(0xffffffffu, m, o);  // half-warp = one child
        const double mR = __shfl_sync(0xffffffffu, m, 16);
        if (lane == 0) {
            const int64_t k = (int64_t)split((double)n, m, mR, seed, tag, d, (uint64_t)i);
            dense[pos] = k;
            dense[pos + R / 2] = n - k;
        }
    }
}

template <typename T2>
cudaError_t dense_levels(const T2* psi, int64_t* dense, int nl, int D, uint64_t seed, uint32_t tag, cudaStream_t st) {
    for (int d = D; d < nl; ++d) {
        const int r = nl - d;  // node range 2^r amplitudes
        const int64_t nn = 1ll << d;
        const unsigned tb = (unsigned)std::min<int64_t>((nn + 255) / 256, 148 * 32);
        const unsigned wb = (unsigned)std::min<int64_t>((nn * 32 + 255) / 256, 148 * 32);
        switch (r) {
            case 8: level_warp<T2, 8><<<wb, 256, 0, st>>>(psi, dense, nl, d, seed, tag); break;
            case 7: level_warp<T2, 4><<<wb, 256, 0, st>>>(psi, dense, nl, d, seed, tag); break;
            case 6: level_warp<T2, 2><<<wb, 256, 0, st>>>(psi, dense, nl, d, seed, tag); break;
            case 5: level_thread<T2, 16><<<tb, 256, 0, st>>>(psi, dense, nl, d, seed, tag); break;
            case 4: level_thread<T2, 8><<<tb, 256, 0, st>>>(psi, dense, nl, d, seed, tag); break;
            case 3: level_thread<T2, 4><<<tb, 256, 0, st>>>(psi, dense, nl, d, seed, tag); break;
            case 2: level_thread<T2, 2><<<tb, 256, 0, st>>>(psi, dense, nl, d, seed, tag); break;
            default: level_thread<T2, 1><<<tb, 256, 0, st>>>(psi, dense, nl, d, seed, tag); break;
        }
    }
    return cudaGetLastError();
}

__global__ void split_parts(const double* __restrict__ masses, int n_parts, int64_t shots, uint64_t seed,
                            int64_t* __restrict__ out) {
    // binary tree over the parts (n_parts a power of two), tag 1, one thread
    if (threadIdx.x || blockIdx.x) return;
    int64_t c[64];
    double m[128];
    const int L = 31 - __clz(n_parts);
    for (int i = 0; i < n_parts; ++i) m[n_parts - 1 + i] = masses[i];
    for (int i = n_parts - 2; i >= 0; --i) m[i] = m[2 * i + 1] + m[2 * i + 2];
    int64_t cur[64];
    cur[0] = shots;
    for (int d = 0; d < L; ++d) {
        const int n = 1 << d;
        for (int i = 0; i < n; ++i) {
            const double mL = m[(2 * n - 1) + 2 * i], mR = m[(2 * n - 1) + 2 * i + 1];
            const int64_t l = (int64_t)split((double)cur[i], mL, mR, seed, 1u, d, (uint64_t)i);
            c[2 * i] = l;
            c[2 * i + 1] = cur[i] - l;
        }
        for (int i = 0; i < 2 * n; ++i) cur[i] = c[i];
    }
    for (int i = 0; i < n_parts; ++i) out[i] = cur[i];
}

// binomial test kernel: out[s] = Binomial(n, p) with node index s (statistical tests)
__global__ void binom_test(double n, double p, uint64_t seed, int64_t count, int64_t* __restrict__ out) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < count; s += (int64_t)gridDim.x * blockDim.x) {
        NodeRng g(seed, 0xffffffu, 63, (uint64_t)s);
        out[s] = (int64_t)binomial(n, p, g);
    }
}

size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

TreeLayout tree_layout(int64_t n_amps) {
    TreeLayout L{};
    L.sb = n_amps < kSubT ? n_amps : kSubT;
    L.n_sub = n_amps / L.sb;
    L.D = 63 - __builtin_clzll((unsigned long long)L.n_sub);
    const int64_t nodes = 2 * L.n_sub - 1;
    size_t scan_b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (const int64_t*)nullptr, (int64_t*)nullptr, L.n_sub + 1);
    size_t o = 0;
    L.off_mass = o; o += al256(nodes * 8);
    L.off_cnt = o; o += al256(nodes * 8);
    L.off_nz = o; o += al256((L.n_sub + 1) * 8);
    L.off_nzpre = o; o += al256((L.n_sub + 1) * 8);
    L.off_cub = o; o += al256(scan_b);
    L.cub_bytes = scan_b;
    L.total = o;
    return L;
}

cudaError_t tree_prepare(const void* psi, int64_t n_amps, int dtype, void* ws, cudaStream_t st) {
    const TreeLayout L = tree_layout(n_amps);
    double* mass = reinterpret_cast<double*>(static_cast<char*>(ws) + L.off_mass);
    double* leaf = mass + (L.n_sub - 1);
    const int64_t threads = L.n_sub * 32;
    const unsigned blocks = (unsigned)((threads + 255) / 256);
    if (dtype == 0) leaf_mass<<<blocks, 256, 0, st>>>(static_cast<const float2*>(psi), L.n_sub, (int)L.sb, leaf);
    else leaf_mass<<<blocks, 256, 0, st>>>(static_cast<const double2*>(psi), L.n_sub, (int)L.sb, leaf);
    for (int d = L.D - 1; d >= 0; --d) {
        const int64_t n = 1ll << d;
        tree_up<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, st>>>(mass, d);
    }
    return cudaGetLastError();
}

const double* tree_total_ptr(const void* ws) {
    return reinterpret_cast<const double*>(static_cast<const char*>(ws) + tree_layout(1).off_mass);
}

cudaError_t tree_draw(const void* psi, int64_t n_amps, int dtype, void* ws, int64_t shots, uint64_t seed, uint32_t tag,
                      int mode, int64_t idx_base, int64_t* out_idx, int64_t* out_cnt, int64_t* n_unique_dev,
                      cudaStream_t st) {
    const TreeLayout L = tree_layout(n_amps);
    char* w = static_cast<char*>(ws);
    const double* mass = reinterpret_cast<const double*>(w + L.off_mass);
    int64_t* cnt = reinterpret_cast<int64_t*>(w + L.off_cnt);
    int64_t* nz = reinterpret_cast<int64_t*>(w + L.off_nz);
    int64_t* nzpre = reinterpret_cast<int64_t*>(w + L.off_nzpre);
    set_root<<<1, 1, 0, st>>>(cnt, shots);
    for (int d = 0; d < L.D; ++d) {
        const int64_t n = 1ll << d;
        tree_down<<<(unsigned)std::min<int64_t>((n + 127) / 128, 148 * 16), 128, 0, st>>>(mass, cnt, d, seed, tag);
    }
    const int64_t* leaf_cnt = cnt + (L.n_sub - 1);
    const unsigned blocks = (unsigned)((L.n_sub * 32 + 255) / 256);
    const int sb = (int)L.sb;
    auto leaf = [&](auto* p) {
        using T2 = std::remove_const_t<std::remove_pointer_t<decltype(p)>>;
        if (mode == 1 && sb == kSubT) {  // level-synchronous below the stored leaves
            const int nl = 63 - __builtin_clzll((unsigned long long)n_amps);
            scatter_leaves<<<(unsigned)std::min<int64_t>((L.n_sub + 255) / 256, 148 * 32), 256, 0, st>>>(
                leaf_cnt, L.n_sub, 8, out_cnt);
            return dense_levels<T2>(p, out_cnt, nl, L.D, seed, tag, st);
        }
        if (mode == 1) {
            tree_leaf<T2, 2><<<blocks, 256, 0, st>>>(p, L.n_sub, sb, L.D, leaf_cnt, seed, tag, idx_base, nullptr,
                                                     nullptr, nullptr, out_cnt);
            return cudaGetLastError();
        }
        tree_leaf<T2, 0><<<blocks, 256, 0, st>>>(p, L.n_sub, sb, L.D, leaf_cnt, seed, tag, idx_base, nz, nullptr,
                                                 nullptr, nullptr);
        cudaMemsetAsync(nz + L.n_sub, 0, 8, st);
        size_t tb = L.cub_bytes;
        cudaError_t e = cub::DeviceScan::ExclusiveSum(w + L.off_cub, tb, nz, nzpre, L.n_sub + 1, st);
        if (e != cudaSuccess) return e;
        tree_leaf<T2, 1><<<blocks, 256, 0, st>>>(p, L.n_sub, sb, L.D, leaf_cnt, seed, tag, idx_base, nullptr, nzpre,
                                                 out_idx, out_cnt);
        if (n_unique_dev) cudaMemcpyAsync(n_unique_dev, nzpre + L.n_sub, 8, cudaMemcpyDeviceToDevice, st);
        return cudaGetLastError();
    };
    if (dtype == 0) return leaf(static_cast<const float2*>(psi));
    return leaf(static_cast<const double2*>(psi));
}

const int64_t* tree_nunique_ptr(const void* ws, int64_t n_amps) {
    const TreeLayout L = tree_layout(n_amps);
    return reinterpret_cast<const int64_t*>(static_cast<const char*>(ws) + L.off_nzpre) + L.n_sub;
}

cudaError_t tree_split_parts(const double* masses_host, int n_parts, int64_t shots, uint64_t seed, void* ws,
                             int64_t* out_host, cudaStream_t st) {
    double* m = static_cast<double*>(ws);  // 64 masses + 64 counts
    int64_t* o = reinterpret_cast<int64_t*>(m + 64);
    cudaError_t e = cudaMemcpyAsync(m, masses_host, n_parts * 8, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    split_parts<<<1, 1, 0, st>>>(m, n_parts, shots, seed, o);
    e = cudaMemcpyAsync(out_host, o, n_parts * 8, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(st);
}

cudaError_t binomial_test(double n, double p, uint64_t seed, int64_t count, int64_t* out, cudaStream_t st) {
    binom_test<<<(unsigned)std::min<int64_t>((count + 255) / 256, 148 * 8), 256, 0, st>>>(n, p, seed, count, out);
    return cudaGetLastError();
}

}  // namespace qg
