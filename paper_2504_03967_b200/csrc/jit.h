// jit.h — circuit-specialised fused-pass kernels.
//
// The interpreter kernel (fused.cu) walks a pass's op words at run time and
// dispatches each through a jump table.  For large states the planner's
// program is instead turned into straight-line PTX per pass (jit.cpp): the
// same op semantics and FP operation order (so the two paths agree bit for
// bit), with every slot, coefficient offset, predicate bit and SMEM / global
// address offset a compile-time constant — no dispatch, no per-op coefficient
// loads and selects, register CX moves as register renames.  The PTX is
// compiled in-process by nvPTXCompiler (thread-safe; plans compile their
// passes on a host thread pool) and loaded with cudaLibraryLoadData.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "desc.h"

namespace qg {

// PTX for one pass (complex64: PassDesc<float>, complex128: PassDesc<double>) on the
// (rb, wb, nbuf) fused-kernel configuration; "" when the pass uses a feature the
// emitter does not cover (the interpreter runs it).  `name` is the entry point.
template <typename Real>
std::string jit_ptx(const PassDesc<Real>& P, int rb, int wb, int nbuf, const std::string& name);
// dynamic SMEM bytes the emitted kernel needs
template <typename Real>
size_t jit_smem_bytes(const PassDesc<Real>& P, int rb, int wb, int nbuf);
// PTX -> sm_100a cubin (nvPTXCompiler); false + log on failure
bool jit_compile(const std::string& ptx, std::vector<char>& cubin, std::string& log);

// a compiled pass (cubin) and its per-device loaded library / kernel / grid;
// shared process-wide through the PTX-keyed cache (jit.cpp)
struct JitModule {
    std::vector<char> cubin;
    struct Dev {
        cudaLibrary_t lib = nullptr;
        cudaKernel_t kern = nullptr;
        int grid = 0;
    };
    std::mutex mu;
    std::vector<Dev> dev;
    ~JitModule();
};

// one pass of a plan: the module, loaded lazily per device
struct JitKernel {
    std::shared_ptr<JitModule> mod;
    std::string name;
    size_t smem = 0;
    int threads = 0;
    bool ok = false;
    std::string err;
};

// P: the pass's PassDesc<float> / PassDesc<double> (the kernel parameter)
cudaError_t launch_jit(JitKernel& k, const void* P, uint64_t n_tiles, void* psi, uint64_t rank_bits, cudaStream_t st);

// Per-plan compilation: worker threads emit + compile the passes in program
// order while the caller may already execute the first ones (wait(i) blocks
// until pass i is ready), so compilation overlaps execution.
struct JitState {
    std::vector<std::unique_ptr<JitKernel>> k;  // index = the plan's d32 index
    std::vector<uint8_t> ready;
    std::mutex mu;
    std::condition_variable cv;
    std::atomic<int64_t> next{0};
    std::vector<std::thread> workers;
    std::atomic<int64_t> n_ok{0}, n_fallback{0};
    std::atomic<int64_t> compile_us{0};   // summed over workers
    int64_t wall_us = 0;                  // start -> last pass compiled
    std::chrono::steady_clock::time_point t0;
    std::string first_error;
    ~JitState();
    JitKernel* wait(int64_t i);           // nullptr: run the interpreter for this pass
    JitKernel* try_get(int64_t i);        // non-blocking: nullptr until pass i is compiled
    // wait for the workers; cancel = stop handing out passes first (passes never
    // compiled stay not-ready: only for plan destruction / rebind)
    void join(bool cancel = false);
};
template <typename Real>
std::shared_ptr<JitState> jit_start(const std::vector<PassDesc<Real>>& descs, int rb, int wb, int nbuf, int threads);
int jit_default_threads();
// passes whose cubin came from the process-wide PTX -> cubin cache (jit.cpp)
int64_t jit_cache_hits();

}  // namespace qg
