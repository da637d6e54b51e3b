// kernels.h — launch entry points of the CUDA translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "desc.h"

namespace qg {

cudaError_t launch_fused(int dtype, int cfg_id, const void* desc, void* psi, uint64_t rank_bits, cudaStream_t st);
cudaError_t launch_gate(int dtype, const GateOp& op, void* psi, int n_local, uint64_t rank_bits, cudaStream_t st);

// uniformly controlled RY (ucry.cu): up to 5 targets per pass
constexpr int kMaxUcryTargets = 5;
struct UcryOp {
    int32_t m, n_t, n_rest, addr_contig;  // address bits, targets, remaining bits, address = contiguous run
    uint8_t addr_pos[40];
    uint8_t tgt_pos[kMaxUcryTargets];
    uint8_t rest_pos[64];
};
int64_t ucry_workspace_bytes(int m, int n_t, int dtype);
cudaError_t launch_ucry(int dtype, void* psi, const UcryOp& op, const double* alpha_dev, void* ws, cudaStream_t st);
cudaError_t launch_qcrank_tally(const int64_t* dense, int m, int nd, int64_t* tot, int64_t* n1, cudaStream_t st);

cudaError_t launch_init_zero(void* psi, int n_local, int dtype, int rank, cudaStream_t st);
cudaError_t launch_init_uniform(void* psi, int n_local, int dtype, int rank, uint64_t mask, cudaStream_t st);
// partial fp64 sums of |a|^2: grid-stride, one double per CTA into `partial`, then
// a single-CTA finish into partial[n_parts]
cudaError_t launch_norm(const void* psi, int64_t n_amps, int dtype, double* partial, int n_parts, cudaStream_t st);
int norm_parts();
cudaError_t launch_probs(const void* psi, int64_t n_amps, int dtype, double* out, cudaStream_t st);

// sampler (see reduce.cu for the layout of the workspace)
int64_t sample_workspace_bytes(int64_t n_amps, int64_t shots);
cudaError_t sample_prefix(const void* psi, int64_t n_amps, int dtype, void* ws, cudaStream_t st, double* total_dev);
cudaError_t sample_draw(const void* psi, int64_t n_amps, int dtype, int64_t shots, uint64_t seed,
                        const double* uniforms, void* ws, int64_t* out_idx, int64_t* out_cnt, cudaStream_t st,
                        int64_t* n_unique_dev);
const double* sample_total_ptr(const void* ws, int64_t n_amps);
const int64_t* sample_nunique_ptr(const void* ws, int64_t n_amps, int64_t shots);

// tree (binomial-split) sampler, tree.cu
struct TreeLayout {
    int64_t sb, n_sub;
    int D;
    size_t off_mass, off_cnt, off_nz, off_nzpre, off_cub, cub_bytes, total;
};
TreeLayout tree_layout(int64_t n_amps);
cudaError_t tree_prepare(const void* psi, int64_t n_amps, int dtype, void* ws, cudaStream_t st);
const double* tree_total_ptr(const void* ws);
// mode 0: (index, count) of the outcomes with a count, ascending; mode 1: dense counts
cudaError_t tree_draw(const void* psi, int64_t n_amps, int dtype, void* ws, int64_t shots, uint64_t seed, uint32_t tag,
                      int mode, int64_t idx_base, int64_t* out_idx, int64_t* out_cnt, int64_t* n_unique_dev,
                      cudaStream_t st);
const int64_t* tree_nunique_ptr(const void* ws, int64_t n_amps);
cudaError_t tree_split_parts(const double* masses_host, int n_parts, int64_t shots, uint64_t seed, void* ws,
                             int64_t* out_host, cudaStream_t st);
cudaError_t binomial_test(double n, double p, uint64_t seed, int64_t count, int64_t* out, cudaStream_t st);

}  // namespace qg
