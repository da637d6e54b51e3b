/*
 * qgear_b200.h — C ABI of libqgear_b200.so, the B200-native executor for the
 * Q-Gear state-vector hot path (arXiv 2504.03967).
 *
 * The reference has no FFI: its executor is pure Python/numpy
 * (/root/reference/pkg/src/qgear/statevec.py, partition.py).  Each entry
 * point below names the reference function/loop it replaces; the Python
 * package paper_2504_03967_b200 binds them with ctypes and keeps the
 * reference's Python signatures on top.
 *
 * Conventions (Appendix A of SURVEY.md):
 *   - qubit k is bit k of the basis index (statevec.py:5-8);
 *   - a state (or one rank's shard) is a contiguous device array of 2^n_local
 *     complex amplitudes, interleaved (re, im): float pairs for
 *     QG_DTYPE_C64 ("fp32", statevec.py:34) or double pairs for QG_DTYPE_C128
 *     ("fp64");
 *   - gate_type rows are (kind, control or -1, target) int32, gate_param is
 *     float64 (ir.py:281-303); kinds H=0 RX=1 RY=2 RZ=3 CX=4 CR1=5
 *     MEASURE=6 (ir.py:31-40);
 *   - all device pointers are plain CUDA device pointers, `stream` is a
 *     cudaStream_t (NULL = legacy default stream);
 *   - every function returns QG_OK (0) or a negative QG_E_* code; the message
 *     of the last failure on the calling thread is qg_last_error().
 */
#ifndef QGEAR_B200_H
#define QGEAR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QG_ABI_VERSION 1

/* status codes -> Python exceptions (paper_2504_03967_b200/errors.py) */
#define QG_OK 0
#define QG_E_INVALID_ARG -1          /* ValueError */
#define QG_E_INDEX_OUT_OF_RANGE -2   /* IndexOutOfRangeError   statevec.py:149-160 */
#define QG_E_SELF_PAIR -3            /* SelfPairError          statevec.py:159-160 */
#define QG_E_MEASURE_MID_CIRCUIT -4  /* MeasureMidCircuitError statevec.py:187-197 */
#define QG_E_TOO_MANY_QUBITS -5      /* TooManyQubitsError     statevec.py:89-91 */
#define QG_E_UNNORMALIZED -6         /* UnnormalizedStateError statevec.py:226-228 */
#define QG_E_BAD_WORKER_COUNT -7     /* BadWorkerCountError    partition.py:82-86 */
#define QG_E_CORRUPT_TENSOR -8       /* CorruptTensorError     ir.py:264-273, 339-345 */
#define QG_E_PROTOCOL -9             /* ProtocolViolationError partition.py:168-173 */
#define QG_E_CUDA -10                /* CUDA runtime / launch failure */
#define QG_E_NONFINITE_PARAM -11     /* NonFiniteParamError */
#define QG_E_INVALID_GATE -12        /* InvalidGateError */
#define QG_E_OUT_OF_MEMORY -13
#define QG_E_CONTAINER_FORMAT -14    /* ContainerFormatError   container.py:87-115 */

#define QG_DTYPE_C64 0
#define QG_DTYPE_C128 1

typedef struct qg_plan qg_plan;

typedef struct {
    int32_t dtype;            /* QG_DTYPE_C64 / QG_DTYPE_C128 */
    int32_t log2_ranks;       /* number of global (sharded) qubits; 0 = one device */
    int32_t fuse;             /* 1 = fused multi-gate passes (default); 0 = one kernel per gate */
    int32_t tile_qubits;      /* 0 = auto; else force the tile width k of fused passes */
    int32_t max_stages;       /* 0 = auto; register stages per pass (SMEM transposes + 1) */
    int32_t max_cost;         /* 0 = auto; per-amplitude instruction budget of one pass */
    int32_t kernel_cfg;       /* 0 = auto; else 1 + id of the fused-kernel configuration (tuning) */
    int32_t jit;              /* circuit-specialised pass kernels (complex64): 0 = auto (shards >= 2^31
                                 amplitudes: on; 2^26..2^30: tiered, compiled in the background while
                                 the interpreter runs), 1 = on, -1 = off (the interpreter runs every pass) */
    int32_t low_qubits;       /* 0 = auto; else the lowest qubits every fused tile contains (>= 5 on
                                 large shards): contiguous runs of 2^low_qubits amplitudes per HBM access */
    int32_t reserved[3];
} qg_plan_opts;

typedef struct {
    int64_t n_body_gates;     /* live gates before the trailing MEASURE block */
    int64_t n_passes;         /* fused-pass (or single-gate) kernel launches per execute */
    int64_t n_segments;       /* passes between two remaps = n_remaps + 1 */
    int64_t n_remaps;         /* qubit-remap all-to-alls (multi-rank only) */
    int64_t n_ops;            /* register-level ops after fusion */
    int64_t n_stages;         /* total register stages over all passes */
    int32_t tile_qubits;      /* k of the fused kernel chosen */
    int32_t n_local;          /* qubits per shard */
    int32_t n_qubits;
    int32_t dtype;
    int64_t param_bytes;      /* kernel-parameter bytes sent per execute (the program, host -> device) */
    int64_t n_cxm;            /* register CX moves the kernel executes (all other register CX gates are
                                 folded into transpose addresses) */
} qg_plan_info;

/* one qubit-remap between segment `seg` and `seg + 1`: physical local
 * positions n_local-s .. n_local-1 swap with the global positions in
 * `global_pos[0..s-1]` (same order). */
typedef struct {
    int32_t s;
    int32_t global_pos[8];
    int32_t local_pos[8];
} qg_remap;

typedef struct {
    double pass_ms;           /* summed CUDA-event time of fused-pass launches (0 if not timed) */
    int64_t pass_launches;    /* kernels launched by qg_plan_execute*, this call */
    int64_t bytes_moved;      /* algorithmic HBM bytes of those launches (2 x shard bytes each) */
} qg_exec_stats;

/* ---- planner: replaces the per-gate dispatch loop statevec.py:207-208 and the
 *      per-gate LOCAL/EXCHANGE tagging partition.py:100-109 ---------------- */
int qg_plan_create(const int32_t* gate_type, const double* gate_param, int64_t n_gates,
                   int32_t n_qubits, const qg_plan_opts* opts, qg_plan** out);
int qg_plan_destroy(qg_plan* plan);

/* Circuit-specialised pass kernels (jit != -1): each fused pass of a complex64
 * plan is emitted as straight-line PTX and compiled on host threads right after
 * qg_plan_create returns; execution waits per pass, so compilation overlaps the
 * first passes.  Status of that compilation (wait = 1 blocks until done). */
typedef struct {
    int64_t n_passes;         /* fused passes in the plan */
    int64_t n_jit;            /* compiled (these run the specialised kernel) */
    int64_t n_fallback;       /* not covered by the emitter: the interpreter runs them */
    int64_t n_pending;
    double compile_ms_sum;    /* emit + compile time summed over passes */
    double compile_ms_wall;   /* plan creation -> last pass compiled */
    int32_t threads;
    int32_t enabled;          /* 0 off, 1 JIT (execution waits per pass), 2 tiered: compiled in the
                                 background, passes run on the interpreter until their kernel is ready */
} qg_jit_status;
int qg_plan_jit_status(const qg_plan* plan, int32_t wait, qg_jit_status* out);
/* the PTX emitted for fused pass `pass_index` (running index over the plan's fused
 * passes); *len = bytes needed (excluding NUL); writes at most cap bytes */
int qg_plan_pass_ptx(const qg_plan* plan, int64_t pass_index, char* buf, int64_t cap, int64_t* len);
/* batched parameter sets (CircuitSet circuits that share one gate structure):
 * new gate_param (n_gates >= the plan's body gates, same order as at create)
 * for the same gate_type; re-emits each pass from its stored schedule (no
 * rescheduling) and rebuilds the device program.  Same errors as create for
 * the parameters (QG_E_NONFINITE_PARAM). */
int qg_plan_rebind(qg_plan* plan, const double* gate_param, int64_t n_gates);
int qg_plan_get_info(const qg_plan* plan, qg_plan_info* out);
int qg_plan_get_remap(const qg_plan* plan, int64_t remap_index, qg_remap* out);
/* logical qubit q sits at physical position phys_of_logical[q] after the last
 * segment (identity unless remaps ran); n_qubits entries */
int qg_plan_get_final_map(const qg_plan* plan, int32_t* phys_of_logical);
/* debug/test export of the fused program at kernel-op granularity, exactly
 * what the fused kernel executes (slot coordinates, desc.h):
 *   rec[i*8 + ...] = {pass, stage, kind, t, c, cmask, qmask, mat}
 *   kind 0 RD / 1 CD (2x2 on slot pairs {p, p^t}, logical |0> member where
 *   parity(c & p ^ c & F) = 0; mats row = complex 2x2), 2 PH (phase e where
 *   parity(t & (p ^ F)) = 1, thread predicate cmask), 3 CXM (slot move along t
 *   where slot bit c = 1), 4 PH2 (phase on |11> of slot bits t, c), 5 XF (flip
 *   vector t where cmask holds), 6 TPH (thread phase v0 / v1 by qmask, where cmask
 *   holds), 100/101 single-gate kernel (GateOp kind 0/1), 200 stage header
 *   (t = register bits, c = packed out vectors 6 bits each, mats row = physical
 *   qubit of each register bit).
 * Call with NULL buffers to get the counts. */
int qg_plan_export(const qg_plan* plan, int64_t* rec, int64_t* n_rec, double* mats, int64_t* n_mats);

/* ---- execution ------------------------------------------------------------ */
/* init_zero_state (statevec.py:81-94) for one shard: amplitude 0 = 1 on rank 0 */
int qg_state_init_zero(void* state, int32_t n_local, int32_t dtype, int32_t rank, void* stream);
/* H on every qubit of qubit_mask (global positions) applied to |0...0>, in one
 * write pass: amplitude 2^(-popcount(mask)/2) where the global index has no bit
 * outside the mask (QCrank's address-register preparation, qcrank.simulate) */
int qg_state_init_uniform(void* state, int32_t n_local, int32_t dtype, uint64_t qubit_mask, int32_t rank,
                          void* stream);
/* run one segment of the plan (all passes on one device): replaces statevec.py:207-208
 * (and the per-worker loop partition.py:265-274 for the LOCAL part) */
int qg_plan_execute_segment(const qg_plan* plan, int64_t segment, void* state, int32_t rank,
                            void* stream, int32_t timed, qg_exec_stats* stats);
/* all segments back to back (single device, log2_ranks == 0) */
int qg_plan_execute(const qg_plan* plan, void* state, void* stream, int32_t timed, qg_exec_stats* stats);

/* ---- the reference's array kernels (statevec.py:115-144), one launch each ----- */
/* u = 2x2 complex row-major as 8 doubles (re00, im00, re01, im01, re10, im10, re11, im11) */
int qg_apply_matrix(void* state, int32_t n_local, int32_t dtype, int32_t target, const double* u, void* stream);
int qg_apply_cx(void* state, int32_t n_local, int32_t dtype, int32_t control, int32_t target, void* stream);
int qg_apply_cr1(void* state, int32_t n_local, int32_t dtype, int32_t control, int32_t target, double lam,
                 void* stream);

/* ---- QCrank data register: uniformly controlled RY --------
 * For every assignment a of the m address qubits (bit k of a = qubit
 * addr_qubits[k]) apply RY(alpha_dev[a * n_targets + j]) to qubit targets[j],
 * j < n_targets <= 5, in one pass.  Equivalent to the Gray-code gate block
 * (2^m RY + 2^m CX per target) that qcrank.build_qcrank_circuit emits; the host
 * collapses that block to this call.  alpha_dev: float64 device array.
 * workspace >= qg_ucry_workspace_bytes (per-address cos/sin table). */
int64_t qg_ucry_workspace_bytes(int32_t m, int32_t n_targets, int32_t dtype);
int qg_apply_ucry(void* state, int32_t n_local, int32_t dtype, const int32_t* addr_qubits, int32_t m,
                  const int32_t* targets, int32_t n_targets, const double* alpha_dev, void* workspace,
                  int64_t workspace_bytes, void* stream);

/* qg_sample (Philox uniforms) without any host synchronisation (CUDA-graph
 * capturable): the norm is written to norm_sq_dev instead of being checked, the
 * number of unique outcomes to n_unique_dev; the caller checks the norm after the
 * stream has run (statevec.CircuitGraph.result). */
int qg_sample_async(const void* state, int64_t n_amps, int32_t dtype, int64_t shots, uint64_t seed,
                    void* workspace, int64_t workspace_bytes, int64_t* out_index_dev, int64_t* out_count_dev,
                    int64_t* n_unique_dev, double* norm_sq_dev, void* stream);
/* QCrank decode tallies from dense per-outcome counts
 * (qg_sample_tree_draw mode 1) of an m-address + n_data-data-qubit state
 * (outcome = address + 2^m * data bits): tot_dev[a] = shots at address a,
 * n1_dev[a * n_data + j] = those with data qubit j = 1; one HBM read. */
int qg_qcrank_tally(const int64_t* dense_counts, int32_t m, int32_t n_data, int64_t* tot_dev, int64_t* n1_dev,
                    void* stream);
/* ---- reductions and sampling (statevec.py:47-50, 215-234) ----------------- */
/* sum |a|^2 in float64; result written to *out_host (synchronises `stream`) */
int qg_norm_sq(const void* state, int64_t n_amps, int32_t dtype, void* workspace, int64_t workspace_bytes,
               double* out_host, void* stream);
/* probs_dev[i] = |a_i|^2 in float64 */
int qg_probabilities(const void* state, int64_t n_amps, int32_t dtype, double* probs_dev, void* stream);

/* Multinomial sampler.  `uniforms_dev` = NULL: counter-based Philox4x32-10
 * uniforms from `seed`; otherwise `shots` caller-supplied uniforms in [0,1)
 * (e.g. numpy default_rng(seed).random(shots), which reproduces the
 * reference's Generator.choice draws).  The norm is checked against
 * `norm_tol` first (QG_E_UNNORMALIZED).  Output: unique outcome indices in
 * increasing order and their counts, n_unique written to *n_unique_host. */
int64_t qg_sample_workspace_bytes(int64_t n_amps, int64_t shots);
int qg_sample(const void* state, int64_t n_amps, int32_t dtype, int64_t shots, uint64_t seed,
              const double* uniforms_dev, double norm_tol, void* workspace, int64_t workspace_bytes,
              int64_t* out_index_dev, int64_t* out_count_dev, int64_t* n_unique_host,
              double* norm_sq_host, void* stream);

/* Tree sampler (tree.cu): the counts of a multinomial draw of `shots` outcomes
 * from |a|^2, generated top-down by binomial splits over the binary tree of
 * the index bits (exactly multinomial; replaces sample_counts statevec.py:221-234
 * when shots are large or the state is sharded).  shots is int64 (< 2^53), the
 * workspace is O(n_amps / 256) (never O(shots)); the result for a given
 * (seed, tag) does not depend on the launch geometry.
 *   prepare: masses of every tree node (one HBM read of the state); *mass_host
 *            = sum |a|^2 (fp64) — the shard mass of a sharded state;
 *   draw:    mode 0: the outcomes with a nonzero count as (index_base + index,
 *            count) pairs in ascending index order, *n_out_host = their number
 *            (capacity >= min(shots, n_amps)); mode 1: dense counts
 *            out_count_dev[n_amps] (capacity >= n_amps), out_index_dev unused.
 *            tag (< 2^24) selects an independent stream (the rank of a shard).
 *            n_out_dev (optional, mode 0): the count also written to device memory,
 *            stream-ordered — with n_out_host NULL the call never synchronises
 *            (CUDA-graph capturable, like prepare with mass_host NULL).
 * A sharded state: every rank prepares, the rank masses are all-gathered, and
 * qg_split_shots (same seed on every rank) splits the shots over the ranks by
 * the same binomial tree (tag 1); each rank then draws its count with tag 2+rank.
 * This path does not check the norm: the caller compares the mass with 1. */
int64_t qg_sample_tree_workspace_bytes(int64_t n_amps);
int qg_sample_tree_prepare(const void* state, int64_t n_amps, int32_t dtype, void* workspace, int64_t workspace_bytes,
                           double* mass_host, void* stream);
int qg_sample_tree_draw(const void* state, int64_t n_amps, int32_t dtype, void* workspace, int64_t workspace_bytes,
                        int64_t shots, uint64_t seed, uint32_t tag, int32_t mode, int64_t index_base,
                        int64_t* out_index_dev, int64_t* out_count_dev, int64_t capacity, int64_t* n_out_host,
                        int64_t* n_out_dev, void* stream);
/* counts_host[r] for r < n_parts (a power of two <= 64) from masses_host[r];
 * workspace: >= 1 KiB of device memory */
int qg_split_shots(const double* masses_host, int32_t n_parts, int64_t shots, uint64_t seed, void* workspace,
                   int64_t workspace_bytes, int64_t* counts_host, void* stream);
/* test hook: out_dev[s] = Binomial(n, p) draws s = 0..count-1 of the sampler's generator */
int qg_binomial_test(double n, double p, uint64_t seed, int64_t count, int64_t* out_dev, void* stream);
/* ---- QGIR1 container (container.py:1-16, 71-115): native parse / write ------
 * qg_qgir1_parse validates a whole file image and reports the byte offsets of
 * its arrays (zero-copy ingest: map the file, pass the int32 / float64 arrays
 * to qg_plan_create); errors (bad magic, truncated, trailing bytes) return
 * QG_E_CONTAINER_FORMAT with the message in qg_container_last_error(). */
typedef struct {
    uint32_t capacity, n_circ, n_meta, pad;
    int64_t headers_off;      /* int32 (n_circ, 3) */
    int64_t gate_type_off;    /* int32 (n_circ, capacity, 3) */
    int64_t gate_param_off;   /* float64 (n_circ, capacity) */
    int64_t meta_off;         /* n_meta x (u32 len, key, u32 len, value) */
    int64_t total_bytes;
} qg_qgir1_info;
int qg_qgir1_parse(const void* buf, int64_t len, qg_qgir1_info* out);
int64_t qg_qgir1_size(uint32_t capacity, uint32_t n_circ, uint32_t n_meta, const int64_t* meta_lens);
/* meta: 2*n_meta strings (key0, value0, key1, ...) in sorted key order, byte lengths in meta_lens */
int qg_qgir1_write(void* buf, int64_t len, uint32_t capacity, uint32_t n_circ, const int32_t* headers,
                   const int32_t* gate_type, const double* gate_param, uint32_t n_meta, const char* const* meta,
                   const int64_t* meta_lens);
const char* qg_container_last_error(void);

const char* qg_last_error(void);
int qg_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QGEAR_B200_H */
