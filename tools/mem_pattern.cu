// HBM microbenchmark of the fused pass's memory structure (dev probe, not product code):
// in-place read + write of a 2^32-amplitude complex64 state through 2^13-amplitude tiles
// with a given tile-bit layout, for several load/store structures.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mem_pattern tools/mem_pattern.cu
//   ./mem_pattern            (prints one line per structure x layout)
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int K = 13;  // tile qubits
struct Layout {
    uint8_t tq[K];       // tile bit -> physical qubit (tq[0..4] = 0..4)
    uint8_t cq[64];      // comp bit -> physical qubit
    int ncomp;
};

__device__ __forceinline__ uint64_t deposit(uint64_t v, const uint8_t* q, int nb) {
    uint64_t r = 0;
    for (int b = 0; b < nb; ++b) r |= ((v >> b) & 1ull) << q[b];
    return r;
}

// S1: thread holds 32 amplitudes; lanes = tile bits 0..4 (one 256 B run per warp access);
// warp w (3 bits) + register r (5 bits) = tile bits 5..12; all loads, then all stores.
template <int MODE>
__global__ void __launch_bounds__(256, 2) s1(float2* psi, const __grid_constant__ Layout L, uint64_t n_tiles) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t roff[32];
    if (threadIdx.x < 32) roff[threadIdx.x] = (uint32_t)deposit((uint64_t)threadIdx.x << 8, L.tq, K);
    __syncthreads();
    const uint32_t lw = (uint32_t)deposit((uint64_t)lane | ((uint64_t)warp << 5), L.tq, 8);
#define loff(r) (lw | roff[r])
    for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const uint64_t base = deposit(t, L.cq, L.ncomp);
        float2 a[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) a[r] = psi[base | loff(r)];
        if (MODE == 1) {  // prefetch the next tile into L2 (one 256 B chunk per thread)
            const uint64_t nt = t + gridDim.x;
            if (nt < n_tiles) {
                const uint64_t nb = deposit(nt, L.cq, L.ncomp) | deposit((uint64_t)threadIdx.x << 5, L.tq, K);
                asm volatile("prefetch.global.L2 [%0];" ::"l"(psi + nb));
            }
        }
#pragma unroll
        for (int r = 0; r < 32; ++r) { a[r].x *= 1.0000001f; a[r].y *= 1.0000001f; }
#pragma unroll
        for (int r = 0; r < 32; ++r) psi[base | loff(r)] = a[r];
    }
}

// S2: 16 B accesses: a thread holds 16 float4 (2 amplitudes each); lanes 0..15 cover one
// 256 B run, lane bit 4 + warp + register = the other 8 tile bits.
__global__ void __launch_bounds__(256, 2) s2(float4* psi4, const __grid_constant__ Layout L, uint64_t n_tiles) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t roff[16];
    if (threadIdx.x < 16) roff[threadIdx.x] = (uint32_t)deposit((uint64_t)threadIdx.x << 9, L.tq, K);
    __syncthreads();
    // amplitude index of float4 element: tile bits 0 = pair member; lanes 0..3 = tile bits 1..4
    const uint32_t lw = (uint32_t)deposit(((uint64_t)(lane & 15) << 1) | ((uint64_t)(lane >> 4) << 5) |
                                          ((uint64_t)warp << 6), L.tq, 9);
    for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const uint64_t base = deposit(t, L.cq, L.ncomp);
        float4 a[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) a[r] = psi4[(base | loff(r)) >> 1];
#pragma unroll
        for (int r = 0; r < 16; ++r) { a[r].x *= 1.0000001f; a[r].w *= 1.0000001f; }
#pragma unroll
        for (int r = 0; r < 16; ++r) psi4[(base | loff(r)) >> 1] = a[r];
    }
}

// S3: S1 with the tile split in two halves: loads of half h+1 overlap stores of half h
// (software pipeline across the tile sequence: load next tile's first half before
// storing the current second half).
__global__ void __launch_bounds__(256, 2) s3(float2* psi, const __grid_constant__ Layout L, uint64_t n_tiles) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t roff[32];
    if (threadIdx.x < 32) roff[threadIdx.x] = (uint32_t)deposit((uint64_t)threadIdx.x << 8, L.tq, K);
    __syncthreads();
    const uint32_t lw = (uint32_t)deposit((uint64_t)lane | ((uint64_t)warp << 5), L.tq, 8);
#define loff(r) (lw | roff[r])
    uint64_t t = blockIdx.x;
    if (t >= n_tiles) return;
    float2 a[32];
    uint64_t base = deposit(t, L.cq, L.ncomp);
#pragma unroll
    for (int r = 0; r < 32; ++r) a[r] = psi[base | loff(r)];
    for (;;) {
#pragma unroll
        for (int r = 0; r < 32; ++r) { a[r].x *= 1.0000001f; a[r].y *= 1.0000001f; }
        const uint64_t nt = t + gridDim.x;
        const bool more = nt < n_tiles;
        const uint64_t nbase = more ? deposit(nt, L.cq, L.ncomp) : 0;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
            psi[base | loff(r)] = a[r];
            if (more) a[r] = psi[nbase | loff(r)];
        }
        if (!more) break;
        t = nt;
        base = nbase;
    }
}

__global__ void fill(float2* p, uint64_t n) {  // incompressible contents
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t h = i * 0x9E3779B97F4A7C15ull;
        h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
        p[i] = make_float2((float)(uint32_t)h * 2.3e-10f - 0.5f, (float)(uint32_t)(h >> 32) * 2.3e-10f - 0.5f);
    }
}

// reference: grid-stride in-place contiguous 16 B read-modify-write
__global__ void inplace(float4* p, uint64_t n4) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
        float4 v = p[i];
        v.x *= 1.0000001f;
        p[i] = v;
    }
}

static Layout make(const std::vector<int>& free8, int n) {
    Layout L{};
    std::vector<char> in(n, 0);
    for (int b = 0; b < 5; ++b) { L.tq[b] = (uint8_t)b; in[b] = 1; }
    for (int j = 0; j < 8; ++j) { L.tq[5 + j] = (uint8_t)free8[j]; in[free8[j]] = 1; }
    int c = 0;
    for (int q = 0; q < n; ++q) if (!in[q]) L.cq[c++] = (uint8_t)q;
    L.ncomp = c;
    return L;
}

int main(int argc, char** argv) {
    const int n = 32;
    const uint64_t N = 1ull << n, bytes = N * 8;
    float2* psi;
    CK(cudaMalloc(&psi, bytes));
    CK(cudaMemset(psi, 0, bytes));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    if (std::getenv("MP_RANDOM")) { fill<<<sms * 8, 256>>>(psi, N); CK(cudaDeviceSynchronize()); }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Lay { const char* name; std::vector<int> f; };
    std::vector<Lay> lays = {
        {"contig", {5, 6, 7, 8, 9, 10, 11, 12}},
        {"plan", {5, 6, 9, 14, 18, 22, 27, 30}},
        {"plan2", {8, 11, 13, 17, 20, 24, 26, 29}},
        {"hi8", {24, 25, 26, 27, 28, 29, 30, 31}},
    };
    auto timeit = [&](auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int i = 0; i < 5; ++i) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        return best;
    };
    const double gb = 2.0 * bytes / 1e9;
    if (std::getenv("MP_SMEM")) {  // s3 / s1 with dynamic shared memory reserved per CTA (shrinks L1)
        CK(cudaFuncSetAttribute(s3, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CK(cudaFuncSetAttribute(s1<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        const Layout L = make({6, 12, 14, 16, 18, 20, 22, 27}, n);
        for (int kb : {0, 16, 32, 48, 64, 70, 80, 96}) {
            const size_t sm = (size_t)kb * 1024;
            const float a3 = timeit([&] { s3<<<sms * 2, 256, sm>>>(psi, L, N >> K); });
            const float a1 = timeit([&] { s1<0><<<sms * 2, 256, sm>>>(psi, L, N >> K); });
            std::printf("smem %3d KB/CTA: s3 %.3f ms s1 %.3f ms\n", kb, a3, a1);
        }
        CK(cudaGetLastError());
        return 0;
    }
    if (argc > 1) {  // tile layouts of a plan ("tile q0 .. q12" lines): sum over the passes
        FILE* f = std::fopen(argv[1], "r");
        if (!f) return 1;
        std::vector<std::vector<int>> tiles;
        char w[16];
        while (std::fscanf(f, "%15s", w) == 1) {
            std::vector<int> t(K);
            for (int j = 0; j < K; ++j) if (std::fscanf(f, "%d", &t[j]) != 1) return 1;
            tiles.push_back(std::vector<int>(t.begin() + 5, t.end()));
        }
        std::fclose(f);
        double t1 = 0, t3 = 0, t2 = 0;
        std::vector<float> per;
        for (const auto& fr : tiles) {
            const Layout L = make(fr, n);
            const uint64_t nt = N >> K;
            const float a1 = timeit([&] { s1<0><<<sms * 2, 256>>>(psi, L, nt); });
            const float a3 = timeit([&] { s3<<<sms * 2, 256>>>(psi, L, nt); });
            const float a2 = timeit([&] { s2<<<sms * 2, 256>>>((float4*)psi, L, nt); });
            t1 += a1; t3 += a3; t2 += a2;
            std::printf("tile");
            for (int q : fr) std::printf(" %d", q);
            std::printf("  s1 %.3f s3 %.3f s2 %.3f\n", a1, a3, a2);
        }
        std::printf("plan %zu passes: s1 %.1f ms (%.3f / pass) s3 %.1f ms (%.3f / pass) s2 %.1f ms (%.3f / pass)\n",
                    tiles.size(), t1, t1 / tiles.size(), t3, t3 / tiles.size(), t2, t2 / tiles.size());
        return 0;
    }
    {
        const float ms = timeit([&] { inplace<<<sms * 8, 256>>>((float4*)psi, bytes / 16); });
        std::printf("inplace-contig-16B          %8.3f ms %7.0f GB/s\n", ms, gb / ms * 1e3);
    }
    for (const auto& ly : lays) {
        const Layout L = make(ly.f, n);
        const uint64_t nt = N >> K;
        for (int occ : {1, 2}) {
            const int grid = sms * occ;
            float ms = timeit([&] { s1<0><<<grid, 256>>>(psi, L, nt); });
            std::printf("s1   %-7s ctas/sm %d      %8.3f ms %7.0f GB/s\n", ly.name, occ, ms, gb / ms * 1e3);
            ms = timeit([&] { s1<1><<<grid, 256>>>(psi, L, nt); });
            std::printf("s1pf %-7s ctas/sm %d      %8.3f ms %7.0f GB/s\n", ly.name, occ, ms, gb / ms * 1e3);
            ms = timeit([&] { s2<<<grid, 256>>>((float4*)psi, L, nt); });
            std::printf("s2   %-7s ctas/sm %d      %8.3f ms %7.0f GB/s\n", ly.name, occ, ms, gb / ms * 1e3);
            ms = timeit([&] { s3<<<grid, 256>>>(psi, L, nt); });
            std::printf("s3   %-7s ctas/sm %d      %8.3f ms %7.0f GB/s\n", ly.name, occ, ms, gb / ms * 1e3);
        }
    }
    CK(cudaGetLastError());
    return 0;
}
