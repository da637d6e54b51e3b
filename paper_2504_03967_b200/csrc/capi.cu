// capi.cu — the extern "C" boundary of libqgear_b200.so (include/qgear_b200.h).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/qgear_b200.h"
#include "jit.h"
#include "kernels.h"
#include "plan.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(QG_E_CUDA, std::string(where) + ": " + cudaGetErrorName(e) + ": " + cudaGetErrorString(e));
}

#define QG_CUDA(call, where)                         \
    do {                                             \
        cudaError_t e_ = (call);                     \
        if (e_ != cudaSuccess) return cuda_fail(e_, where); \
    } while (0)

// Every entry point that launches work on a state makes the state's device the
// current one for the call (a stream of device d only takes launches while d is
// current), restoring the caller's device on return.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(const void* ptr) {
        if (!ptr) return;
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) { cudaGetLastError(); return; }
        if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return;
        int cur = 0;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != a.device && cudaSetDevice(a.device) == cudaSuccess) prev = cur;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// fused-kernel configurations the JIT emitter covers (must match launch_fused:
// complex64 ids >= 4 are the single-buffered ones)
int jit_nbuf(const qg_plan& p) {
    // dev probe QG_DEV_JIT_CFG0: the JIT (single-buffered) also for the 16-warp complex64 tile (id 0)
    static const bool cfg0 = std::getenv("QG_DEV_JIT_CFG0") != nullptr;
    if (cfg0 && p.dtype == QG_DTYPE_C64 && p.cfg.id <= 1) return 1;
    if (cfg0 && p.dtype == QG_DTYPE_C128 && p.cfg.id == 0) return 1;
    return p.dtype == QG_DTYPE_C64 ? (p.cfg.id >= 4 ? 1 : 2) : (p.cfg.id == 3 ? 1 : 2);
}

// 0 = interpreter only, 1 = JIT (execution waits for each pass's kernel), 2 = tiered:
// passes compile in the background and run on the interpreter until their kernel is
// ready (the two produce bit-identical states, test_gpu_jit.py); the process-wide
// cubin cache makes every later plan of the same circuit start fully compiled
int jit_wanted(const qg_plan& p, int mode) {
    if (mode < 0 || jit_nbuf(p) != 1) return 0;
    if (p.dtype == QG_DTYPE_C64 ? p.d32.empty() : p.d64.empty()) return 0;
    if (mode > 0) return 1;
    if (p.dtype == QG_DTYPE_C128) return p.n_local >= 30 ? 1 : (p.n_local >= 26 ? 2 : 0);  // same bytes as c64 + 1
    // auto: shards large enough that a pass takes longer than its share of the
    // compilation (~0.2 s of one host core per pass, spread over the host's cores
    // and overlapped with the execution of the earlier passes): >= 2^31 amplitudes;
    // mid-size shards tier up in the background
    if (p.n_local >= 31) return 1;
    return p.n_local >= 26 ? 2 : 0;
}

void jit_launch(qg_plan& p, int mode) {
    const int w = jit_wanted(p, mode);
    if (!w) return;
    p.jit_blocking = w == 1;
    p.jit_threads = w == 1 ? qg::jit_default_threads() : std::min(4, qg::jit_default_threads());
    p.jit = p.dtype == QG_DTYPE_C64 ? qg::jit_start(p.d32, p.cfg.rb, p.cfg.wb, jit_nbuf(p), p.jit_threads)
                                    : qg::jit_start(p.d64, p.cfg.rb, p.cfg.wb, jit_nbuf(p), p.jit_threads);
}

int check_dtype(int32_t dtype) {
    return (dtype == QG_DTYPE_C64 || dtype == QG_DTYPE_C128) ? QG_OK : fail(QG_E_INVALID_ARG, "dtype must be 0 (c64) or 1 (c128)");
}

int run_segment(const qg_plan* plan, int64_t seg, void* state, int32_t rank, cudaStream_t st, qg_exec_stats* stats) {
    const uint64_t rank_bits = (uint64_t)rank << plan->n_local;
    const auto& passes = plan->segs[seg];
    const auto& idx = plan->desc_index[seg];
    const int64_t shard_bytes = ((int64_t)1 << plan->n_local) * (plan->dtype == QG_DTYPE_C64 ? 8 : 16);
    for (size_t p = 0; p < passes.size(); ++p) {
        cudaError_t e;
        qg::JitKernel* jk = nullptr;
        if (idx[p] >= 0 && plan->jit) jk = plan->jit_blocking ? plan->jit->wait(idx[p]) : plan->jit->try_get(idx[p]);
        if (jk) {
            const void* d = plan->dtype == QG_DTYPE_C64 ? (const void*)&plan->d32[idx[p]] : (const void*)&plan->d64[idx[p]];
            const uint64_t nt = plan->dtype == QG_DTYPE_C64 ? plan->d32[idx[p]].n_tiles : plan->d64[idx[p]].n_tiles;
            e = qg::launch_jit(*jk, d, nt, state, rank_bits, st);
        } else if (idx[p] >= 0) {
            const void* d = plan->dtype == QG_DTYPE_C64 ? (const void*)&plan->d32[idx[p]] : (const void*)&plan->d64[idx[p]];
            e = qg::launch_fused(plan->dtype, plan->cfg.id, d, state, rank_bits, st);
        } else {
            e = qg::launch_gate(plan->dtype, passes[p].gop, state, plan->n_local, rank_bits, st);
        }
        if (e != cudaSuccess) return cuda_fail(e, "pass launch");
        if (stats) {
            stats->pass_launches += 1;
            stats->bytes_moved += 2 * shard_bytes;
        }
    }
    return QG_OK;
}

}  // namespace

extern "C" {

const char* qg_last_error(void) { return g_err.c_str(); }
int qg_abi_version(void) { return QG_ABI_VERSION; }

int qg_plan_create(const int32_t* gate_type, const double* gate_param, int64_t n_gates, int32_t n_qubits,
                   const qg_plan_opts* opts, qg_plan** out) {
    if (!out) return fail(QG_E_INVALID_ARG, "out is NULL");
    *out = nullptr;
    qg_plan_opts o{};
    o.fuse = 1;
    if (opts) o = *opts;
    qg_plan* p = new (std::nothrow) qg_plan();
    if (!p) return fail(QG_E_OUT_OF_MEMORY, "plan allocation failed");
    std::string err;
    int rc;
    try {
        rc = qg::build_plan(gate_type, gate_param, n_gates, n_qubits, o, *p, err);
    } catch (const std::bad_alloc&) {
        rc = QG_E_OUT_OF_MEMORY;
        err = "out of host memory while planning";
    }
    if (rc != QG_OK) {
        delete p;
        return fail(rc, err);
    }
    p->jit_mode = o.jit;
    jit_launch(*p, o.jit);
    *out = p;
    return QG_OK;
}

int qg_plan_rebind(qg_plan* plan, const double* gate_param, int64_t n_gates) {
    if (!plan) return fail(QG_E_INVALID_ARG, "plan is NULL");
    std::string err;
    int rc;
    if (plan->jit) {  // the compile workers read the descriptors being rebuilt
        plan->jit->join(true);
        plan->jit.reset();
    }
    try {
        rc = qg::rebind_plan(*plan, gate_param, n_gates, err);
    } catch (const std::bad_alloc&) {
        rc = QG_E_OUT_OF_MEMORY;
        err = "out of host memory while rebinding";
    }
    if (rc == QG_OK) jit_launch(*plan, plan->jit_mode);
    return rc == QG_OK ? QG_OK : fail(rc, err);
}

int qg_plan_jit_status(const qg_plan* plan, int32_t wait, qg_jit_status* out) {
    if (!plan || !out) return fail(QG_E_INVALID_ARG, "NULL argument");
    std::memset(out, 0, sizeof *out);
    out->n_passes = plan->dtype == QG_DTYPE_C64 ? (int64_t)plan->d32.size() : (int64_t)plan->d64.size();
    if (!plan->jit) return QG_OK;
    qg::JitState& J = *plan->jit;
    if (wait) J.join();
    out->enabled = plan->jit_blocking ? 1 : 2;
    out->threads = plan->jit_threads;
    out->n_jit = J.n_ok.load();
    out->n_fallback = J.n_fallback.load();
    out->n_pending = out->n_passes - out->n_jit - out->n_fallback;
    out->compile_ms_sum = J.compile_us.load() / 1000.0;
    {
        std::lock_guard<std::mutex> lk(J.mu);
        out->compile_ms_wall = J.wall_us / 1000.0;
    }
    return QG_OK;
}

int qg_plan_pass_ptx(const qg_plan* plan, int64_t pass_index, char* buf, int64_t cap, int64_t* len) {
    if (!plan || !len) return fail(QG_E_INVALID_ARG, "NULL argument");
    const int64_t nd = plan->dtype == QG_DTYPE_C64 ? (int64_t)plan->d32.size() : (int64_t)plan->d64.size();
    if (pass_index < 0 || pass_index >= nd) return fail(QG_E_INVALID_ARG, "pass_index out of range");
    const std::string ptx =
        plan->dtype == QG_DTYPE_C64
            ? qg::jit_ptx(plan->d32[pass_index], plan->cfg.rb, plan->cfg.wb, jit_nbuf(*plan), "qg_jit_pass")
            : qg::jit_ptx(plan->d64[pass_index], plan->cfg.rb, plan->cfg.wb, jit_nbuf(*plan), "qg_jit_pass");
    *len = (int64_t)ptx.size();
    if (buf && cap > 0) {
        const int64_t n = std::min<int64_t>(cap - 1, (int64_t)ptx.size());
        std::memcpy(buf, ptx.data(), (size_t)n);
        buf[n] = 0;
    }
    return QG_OK;
}

int qg_plan_destroy(qg_plan* plan) {
    delete plan;
    return QG_OK;
}

int qg_plan_get_info(const qg_plan* plan, qg_plan_info* out) {
    if (!plan || !out) return fail(QG_E_INVALID_ARG, "NULL argument");
    std::memset(out, 0, sizeof(*out));
    out->n_body_gates = plan->n_body;
    for (const auto& s : plan->segs) out->n_passes += (int64_t)s.size();
    out->n_segments = (int64_t)plan->segs.size();
    out->n_remaps = (int64_t)plan->remaps.size();
    out->n_ops = plan->stats.n_ops;
    out->n_stages = plan->stats.n_stages;
    out->tile_qubits = plan->cfg.k();
    out->n_local = plan->n_local;
    out->n_qubits = plan->n;
    out->dtype = plan->dtype;
    out->n_cxm = plan->stats.n_cxm;
    for (size_t s = 0; s < plan->segs.size(); ++s)
        for (size_t p = 0; p < plan->segs[s].size(); ++p)
            out->param_bytes += plan->desc_index[s][p] >= 0
                                    ? (int64_t)(plan->dtype == QG_DTYPE_C64 ? sizeof(qg::PassDesc<float>)
                                                                            : sizeof(qg::PassDesc<double>))
                                    : (int64_t)sizeof(qg::GateOp);
    return QG_OK;
}

int qg_plan_get_remap(const qg_plan* plan, int64_t i, qg_remap* out) {
    if (!plan || !out) return fail(QG_E_INVALID_ARG, "NULL argument");
    if (i < 0 || i >= (int64_t)plan->remaps.size()) return fail(QG_E_INVALID_ARG, "remap index out of range");
    *out = plan->remaps[i];
    return QG_OK;
}

int qg_plan_get_final_map(const qg_plan* plan, int32_t* phys_of_logical) {
    if (!plan || !phys_of_logical) return fail(QG_E_INVALID_ARG, "NULL argument");
    for (int q = 0; q < plan->n; ++q) phys_of_logical[q] = plan->final_phys[q];
    return QG_OK;
}

int qg_plan_export(const qg_plan* plan, int64_t* rec, int64_t* n_rec, double* mats, int64_t* n_mats) {
    if (!plan || !n_rec || !n_mats) return fail(QG_E_INVALID_ARG, "NULL argument");
    int64_t nr = 0, nm = 0, pass_id = 0;
    auto row = [&](int64_t s, int64_t kind, int64_t t, int64_t c, uint64_t cmask, uint64_t qmask, const double* m) {
        if (rec) {
            int64_t* r = rec + 8 * nr;
            r[0] = pass_id; r[1] = s; r[2] = kind; r[3] = t; r[4] = c;
            r[5] = (int64_t)cmask; r[6] = (int64_t)qmask; r[7] = nm;
        }
        if (mats) std::memcpy(mats + 8 * nm, m, 8 * sizeof(double));
        ++nr; ++nm;
    };
    const size_t last_seg = plan->segs.size() - 1;
    for (size_t si = 0; si < plan->segs.size(); ++si) {
        const auto& seg = plan->segs[si];
        for (size_t pi = 0; pi < seg.size(); ++pi) {
            const auto& hp = seg[pi];
            if (hp.fused) {
                for (size_t s = 0; s < hp.stages.size(); ++s) {
                    const auto& st = hp.stages[s];
                    double hdr[8] = {0};
                    int64_t packed = 0;
                    for (size_t b = 0; b < st.reg_tile.size(); ++b) {
                        hdr[b] = hp.tile_q[st.reg_tile[b]];
                        packed |= (int64_t)st.out_vec[b] << (6 * b);
                    }
                    row((int64_t)s, 200, (int64_t)st.reg_tile.size(), packed, 0, 0, hdr);
                    for (const auto& o : st.ops) {
                        double m[8] = {0};
                        if (o.kind == qg::A_RD && hp.scaled_rot) {  // scaled form: M = R / sigma
                            const double k = o.m[1] == 0.0 ? 1.0 : o.m[0], t = o.m[1] == 0.0 ? o.m[0] : 1.0;
                            m[0] = k; m[2] = -t; m[4] = t; m[6] = k;
                        } else if (o.kind == qg::A_RD) {  // the three shears as one real 2x2, complex layout
                            const double a = o.m[0], b = o.m[1];
                            m[0] = 1 + a * b; m[2] = 2 * a + a * a * b; m[4] = b; m[6] = 1 + a * b;
                        } else {
                            std::memcpy(m, o.m, sizeof(m));
                        }
                        int64_t t = o.t, c = o.c;
                        if (o.kind == qg::A_RD || o.kind == qg::A_CD) {  // pair vector V, role vector W
                            const int64_t e = 1ll << o.t, f = o.c >= 0 ? (1ll << o.c) : 0;
                            t = o.form == 2 ? (e | f) : e;
                            c = o.form == 1 ? (e | f) : e;
                        } else if (o.kind == qg::A_PH) {  // role vector W; one row per list factor
                            t = (1ll << o.t) | (o.c >= 0 ? (1ll << o.c) : 0);
                            for (const auto& x : o.ph) {
                                const double e[8] = {x.second.first, x.second.second};
                                row((int64_t)s, o.kind, t, -1, x.first, 0, e);
                            }
                            continue;
                        }
                        if (o.kind == qg::A_XF) {  // one row per list entry
                            for (const auto& x : o.xf) row((int64_t)s, o.kind, (int64_t)x.second, -1, x.first, 0, m);
                            continue;
                        }
                        row((int64_t)s, o.kind, t, c, o.cmask, o.qmask, m);
                    }
                    for (const auto& o : st.tph) row((int64_t)s, qg::A_TPH, -1, -1, o.cmask, o.qmask, o.m);
                    if (s + 1 == hp.stages.size() && hp.rscale != 1.0) {  // the pass's rotation scale
                        const double g[8] = {hp.rscale, 0.0, hp.rscale, 0.0};
                        row((int64_t)s, qg::A_TPH, -1, -1, 0, 0, g);
                    }
                    const bool last = si == last_seg && pi + 1 == seg.size() && s + 1 == hp.stages.size();
                    if (last && (plan->gphase_re != 1.0 || plan->gphase_im != 0.0)) {
                        const double g[8] = {plan->gphase_re, plan->gphase_im, plan->gphase_re, plan->gphase_im};
                        row((int64_t)s, qg::A_TPH, -1, -1, 0, 0, g);
                    }
                }
            } else {
                row(-1, 100 + hp.gop.kind, hp.gop.t, -1, hp.gop.cmask, hp.gop.qmask, hp.gop.m);
            }
            ++pass_id;
        }
        ++pass_id;  // a skipped pass id marks a segment boundary (remap)
    }
    *n_rec = nr;
    *n_mats = nm;
    return QG_OK;
}

int qg_state_init_zero(void* state, int32_t n_local, int32_t dtype, int32_t rank, void* stream) {
    DeviceGuard dg_(state);
    if (int rc = check_dtype(dtype)) return rc;
    if (!state || n_local < 0 || n_local > 40) return fail(QG_E_INVALID_ARG, "bad state / n_local");
    QG_CUDA(qg::launch_init_zero(state, n_local, dtype, rank, (cudaStream_t)stream), "init_zero");
    return QG_OK;
}

int qg_state_init_uniform(void* state, int32_t n_local, int32_t dtype, uint64_t qubit_mask, int32_t rank,
                          void* stream) {
    DeviceGuard dg_(state);
    if (int rc = check_dtype(dtype)) return rc;
    if (!state || n_local < 0 || n_local > 40 || rank < 0) return fail(QG_E_INVALID_ARG, "bad state / n_local / rank");
    if (qubit_mask >> n_local) return fail(QG_E_INDEX_OUT_OF_RANGE, "H-layer qubit outside the shard's local qubits");
    QG_CUDA(qg::launch_init_uniform(state, n_local, dtype, rank, qubit_mask, (cudaStream_t)stream), "init_uniform");
    return QG_OK;
}

int qg_plan_execute_segment(const qg_plan* plan, int64_t segment, void* state, int32_t rank, void* stream,
                            int32_t timed, qg_exec_stats* stats) {
    DeviceGuard dg_(state);
    if (!plan || !state) return fail(QG_E_INVALID_ARG, "NULL argument");
    if (segment < 0 || segment >= (int64_t)plan->segs.size()) return fail(QG_E_INVALID_ARG, "segment out of range");
    if (rank < 0 || rank >= (1 << plan->g)) return fail(QG_E_BAD_WORKER_COUNT, "rank out of range");
    cudaStream_t st = (cudaStream_t)stream;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (stats) std::memset(stats, 0, sizeof(*stats));
    if (timed) {
        QG_CUDA(cudaEventCreate(&e0), "event");
        QG_CUDA(cudaEventCreate(&e1), "event");
        QG_CUDA(cudaEventRecord(e0, st), "event record");
    }
    int rc = run_segment(plan, segment, state, rank, st, stats);
    if (timed) {
        if (rc == QG_OK) {
            cudaEventRecord(e1, st);
            cudaError_t e = cudaEventSynchronize(e1);
            float ms = 0;
            if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
            if (e != cudaSuccess) rc = cuda_fail(e, "timed execute");
            else if (stats) stats->pass_ms = ms;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    return rc;
}

int qg_plan_execute(const qg_plan* plan, void* state, void* stream, int32_t timed, qg_exec_stats* stats) {
    if (!plan || !state) return fail(QG_E_INVALID_ARG, "NULL argument");
    if (plan->g != 0) return fail(QG_E_BAD_WORKER_COUNT, "multi-rank plan: use qg_plan_execute_segment + remaps");
    return qg_plan_execute_segment(plan, 0, state, 0, stream, timed, stats);
}

static int single_gate(void* state, int32_t n_local, int32_t dtype, const qg::GateOp& op, void* stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (!state || n_local < 1 || n_local > 40) return fail(QG_E_INVALID_ARG, "bad state / n_local");
    QG_CUDA(qg::launch_gate(dtype, op, state, n_local, 0, (cudaStream_t)stream), "gate launch");
    return QG_OK;
}

int qg_apply_matrix(void* state, int32_t n_local, int32_t dtype, int32_t target, const double* u, void* stream) {
    DeviceGuard dg_(state);
    if (target < 0 || target >= n_local)
        return fail(QG_E_INDEX_OUT_OF_RANGE, "target " + std::to_string(target) + " out of range for " +
                                                 std::to_string(n_local) + " qubits");
    if (!u) return fail(QG_E_INVALID_ARG, "u is NULL");
    qg::GateOp op{};
    op.kind = 0;
    op.t = target;
    std::memcpy(op.m, u, sizeof(op.m));
    return single_gate(state, n_local, dtype, op, stream);
}

int64_t qg_ucry_workspace_bytes(int32_t m, int32_t n_targets, int32_t dtype) {
    if (m < 0 || m > 34 || n_targets < 1 || n_targets > qg::kMaxUcryTargets) return -1;
    return qg::ucry_workspace_bytes(m, n_targets, dtype);
}

int qg_apply_ucry(void* state, int32_t n_local, int32_t dtype, const int32_t* addr_qubits, int32_t m,
                  const int32_t* targets, int32_t n_targets, const double* alpha_dev, void* workspace,
                  int64_t workspace_bytes, void* stream) {
    DeviceGuard dg_(state);
    if (int rc = check_dtype(dtype)) return rc;
    if (!state || !alpha_dev || !workspace || (m > 0 && !addr_qubits) || !targets)
        return fail(QG_E_INVALID_ARG, "NULL argument");
    if (n_targets < 1 || n_targets > qg::kMaxUcryTargets)
        return fail(QG_E_INVALID_ARG, "n_targets must be in [1, 5]");
    if (m < 0 || m > 34 || m + n_targets > n_local) return fail(QG_E_INVALID_ARG, "bad address register size");
    if (workspace_bytes < qg::ucry_workspace_bytes(m, n_targets, dtype))
        return fail(QG_E_INVALID_ARG, "workspace too small");
    std::vector<int> used(n_local, 0);
    qg::UcryOp op{};
    op.m = m;
    op.n_t = n_targets;
    auto take = [&](int q) -> int {
        if (q < 0 || q >= n_local)
            return fail(QG_E_INDEX_OUT_OF_RANGE, "qubit " + std::to_string(q) + " out of range for " +
                                                     std::to_string(n_local) + " qubits");
        if (used[q]) return fail(QG_E_SELF_PAIR, "qubit " + std::to_string(q) + " listed twice");
        used[q] = 1;
        return QG_OK;
    };
    op.addr_contig = 1;
    for (int k = 0; k < m; ++k) {
        if (int rc = take(addr_qubits[k])) return rc;
        op.addr_pos[k] = (uint8_t)addr_qubits[k];
        if (k > 0 && addr_qubits[k] != addr_qubits[k - 1] + 1) op.addr_contig = 0;
    }
    if (m == 0) op.addr_pos[0] = 0;
    for (int j = 0; j < n_targets; ++j) {
        if (int rc = take(targets[j])) return rc;
        op.tgt_pos[j] = (uint8_t)targets[j];
    }
    for (int q = 0; q < n_local; ++q)
        if (!used[q]) op.rest_pos[op.n_rest++] = (uint8_t)q;
    QG_CUDA(qg::launch_ucry(dtype, state, op, alpha_dev, workspace, (cudaStream_t)stream), "ucry launch");
    return QG_OK;
}

static int check_pair(int32_t n, int32_t c, int32_t t) {
    for (int q : {c, t})
        if (q < 0 || q >= n)
            return fail(QG_E_INDEX_OUT_OF_RANGE, "qubit " + std::to_string(q) + " out of range for " +
                                                     std::to_string(n) + " qubits");
    if (c == t) return fail(QG_E_SELF_PAIR, "control == target == " + std::to_string(c));
    return QG_OK;
}

int qg_apply_cx(void* state, int32_t n_local, int32_t dtype, int32_t control, int32_t target, void* stream) {
    DeviceGuard dg_(state);
    if (int rc = check_pair(n_local, control, target)) return rc;
    qg::GateOp op{};
    op.kind = 0;
    op.t = target;
    op.cmask = 1ull << control;
    op.m[2] = 1.0;  // [[0,1],[1,0]]
    op.m[4] = 1.0;
    return single_gate(state, n_local, dtype, op, stream);
}

int qg_apply_cr1(void* state, int32_t n_local, int32_t dtype, int32_t control, int32_t target, double lam,
                 void* stream) {
    DeviceGuard dg_(state);
    if (int rc = check_pair(n_local, control, target)) return rc;
    qg::GateOp op{};
    op.kind = 0;
    op.t = target;
    op.cmask = 1ull << control;
    op.m[0] = 1.0;
    op.m[6] = std::cos(lam);
    op.m[7] = std::sin(lam);
    return single_gate(state, n_local, dtype, op, stream);
}

int qg_norm_sq(const void* state, int64_t n_amps, int32_t dtype, void* workspace, int64_t workspace_bytes,
               double* out_host, void* stream) {
    DeviceGuard dg_(state);
    if (int rc = check_dtype(dtype)) return rc;
    const int parts = qg::norm_parts();
    if (!state || !workspace || !out_host || n_amps < 1) return fail(QG_E_INVALID_ARG, "NULL argument");
    if (workspace_bytes < (int64_t)(parts + 1) * 8) return fail(QG_E_INVALID_ARG, "workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    double* part = static_cast<double*>(workspace);
    QG_CUDA(qg::launch_norm(state, n_amps, dtype, part, parts, st), "norm");
    QG_CUDA(cudaMemcpyAsync(out_host, part + parts, sizeof(double), cudaMemcpyDeviceToHost, st), "norm copy");
    QG_CUDA(cudaStreamSynchronize(st), "norm sync");
    return QG_OK;
}

int qg_probabilities(const void* state, int64_t n_amps, int32_t dtype, double* probs_dev, void* stream) {
    DeviceGuard dg_(state);
    if (int rc = check_dtype(dtype)) return rc;
    if (!state || !probs_dev || n_amps < 1) return fail(QG_E_INVALID_ARG, "NULL argument");
    QG_CUDA(qg::launch_probs(state, n_amps, dtype, probs_dev, (cudaStream_t)stream), "probabilities");
    return QG_OK;
}

int64_t qg_sample_workspace_bytes(int64_t n_amps, int64_t shots) {
    if (n_amps < 1 || shots < 0) return -1;
    return qg::sample_workspace_bytes(n_amps, shots);
}

int qg_sample(const void* state, int64_t n_amps, int32_t dtype, int64_t shots, uint64_t seed,
              const double* uniforms_dev, double norm_tol, void* workspace, int64_t workspace_bytes,
              int64_t* out_index_dev, int64_t* out_count_dev, int64_t* n_unique_host, double* norm_sq_host,
              void* stream) {
    DeviceGuard dg_(state);
    if (int rc = check_dtype(dtype)) return rc;
    if (shots < 1) return fail(QG_E_INVALID_ARG, "shots must be >= 1, got " + std::to_string(shots));
    if (shots > (int64_t)INT32_MAX) return fail(QG_E_INVALID_ARG, "shots > 2^31-1 not supported by this sampler");
    if (!state || !workspace || !out_index_dev || !out_count_dev || !n_unique_host || n_amps < 1 ||
        (n_amps & (n_amps - 1)))
        return fail(QG_E_INVALID_ARG, "bad sampler arguments");
    if (workspace_bytes < qg::sample_workspace_bytes(n_amps, shots)) return fail(QG_E_INVALID_ARG, "workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    QG_CUDA(qg::sample_prefix(state, n_amps, dtype, workspace, st, nullptr), "sample prefix");
    double total = 0;
    QG_CUDA(cudaMemcpyAsync(&total, qg::sample_total_ptr(workspace, n_amps), sizeof(double), cudaMemcpyDeviceToHost, st),
            "norm copy");
    QG_CUDA(cudaStreamSynchronize(st), "sample sync");
    if (norm_sq_host) *norm_sq_host = total;
    if (!(std::fabs(total - 1.0) <= norm_tol)) {  // statevec.py:226-228 (NaN fails too)
        char buf[96];
        std::snprintf(buf, sizeof(buf), "norm^2 = %.17g outside tolerance", total);
        return fail(QG_E_UNNORMALIZED, buf);
    }
    int64_t* nu = const_cast<int64_t*>(qg::sample_nunique_ptr(workspace, n_amps, shots));
    QG_CUDA(qg::sample_draw(state, n_amps, dtype, shots, seed, uniforms_dev, workspace, out_index_dev, out_count_dev, st,
                            nu),
            "sample draw");
    QG_CUDA(cudaMemcpyAsync(n_unique_host, nu, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "nunique copy");
    QG_CUDA(cudaStreamSynchronize(st), "sample sync");
    return QG_OK;
}

int qg_qcrank_tally(const int64_t* dense_counts, int32_t m, int32_t n_data, int64_t* tot_dev, int64_t* n1_dev,
                    void* stream) {
    DeviceGuard dg_(dense_counts);
    if (!dense_counts || !tot_dev || !n1_dev || m < 0 || n_data < 1 || n_data > 16 || m + n_data > 62)
        return fail(QG_E_INVALID_ARG, "bad qcrank tally arguments");
    QG_CUDA(qg::launch_qcrank_tally(dense_counts, m, n_data, tot_dev, n1_dev, (cudaStream_t)stream), "qcrank tally");
    return QG_OK;
}

int qg_sample_async(const void* state, int64_t n_amps, int32_t dtype, int64_t shots, uint64_t seed,
                    void* workspace, int64_t workspace_bytes, int64_t* out_index_dev, int64_t* out_count_dev,
                    int64_t* n_unique_dev, double* norm_sq_dev, void* stream) {
    DeviceGuard dg_(state);
    if (int rc = check_dtype(dtype)) return rc;
    if (shots < 1 || shots > (int64_t)INT32_MAX) return fail(QG_E_INVALID_ARG, "shots must be in [1, 2^31)");
    if (!state || !workspace || !out_index_dev || !out_count_dev || !n_unique_dev || !norm_sq_dev || n_amps < 1 ||
        (n_amps & (n_amps - 1)))
        return fail(QG_E_INVALID_ARG, "bad sampler arguments");
    if (workspace_bytes < qg::sample_workspace_bytes(n_amps, shots)) return fail(QG_E_INVALID_ARG, "workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    QG_CUDA(qg::sample_prefix(state, n_amps, dtype, workspace, st, nullptr), "sample prefix");
    QG_CUDA(cudaMemcpyAsync(norm_sq_dev, qg::sample_total_ptr(workspace, n_amps), sizeof(double),
                            cudaMemcpyDeviceToDevice, st), "norm copy");
    QG_CUDA(qg::sample_draw(state, n_amps, dtype, shots, seed, nullptr, workspace, out_index_dev, out_count_dev, st,
                            n_unique_dev),
            "sample draw");
    return QG_OK;
}

// ---- tree (binomial-split) sampler --------------------------------------------
int64_t qg_sample_tree_workspace_bytes(int64_t n_amps) {
    if (n_amps < 1 || (n_amps & (n_amps - 1))) return -1;
    return (int64_t)qg::tree_layout(n_amps).total;
}

int qg_sample_tree_prepare(const void* state, int64_t n_amps, int32_t dtype, void* workspace, int64_t workspace_bytes,
                           double* mass_host, void* stream) {
    DeviceGuard dg_(state);
    if (int rc = check_dtype(dtype)) return rc;
    if (!state || !workspace || n_amps < 1 || (n_amps & (n_amps - 1)))
        return fail(QG_E_INVALID_ARG, "bad sampler arguments");
    if (workspace_bytes < qg_sample_tree_workspace_bytes(n_amps)) return fail(QG_E_INVALID_ARG, "workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    QG_CUDA(qg::tree_prepare(state, n_amps, dtype, workspace, st), "tree prepare");
    if (mass_host) {
        QG_CUDA(cudaMemcpyAsync(mass_host, qg::tree_total_ptr(workspace), 8, cudaMemcpyDeviceToHost, st), "mass copy");
        QG_CUDA(cudaStreamSynchronize(st), "tree sync");
    }
    return QG_OK;
}

int qg_sample_tree_draw(const void* state, int64_t n_amps, int32_t dtype, void* workspace, int64_t workspace_bytes,
                        int64_t shots, uint64_t seed, uint32_t tag, int32_t mode, int64_t index_base,
                        int64_t* out_index_dev, int64_t* out_count_dev, int64_t capacity, int64_t* n_out_host,
                        int64_t* n_out_dev, void* stream) {
    DeviceGuard dg_(state);
    if (int rc = check_dtype(dtype)) return rc;
    if (shots < 0 || shots >= (1ll << 53)) return fail(QG_E_INVALID_ARG, "shots must be in [0, 2^53)");
    if (!state || !workspace || !out_count_dev || n_amps < 1 || (n_amps & (n_amps - 1)) || (mode != 0 && mode != 1) ||
        tag > 0xffffffu)
        return fail(QG_E_INVALID_ARG, "bad sampler arguments");
    if (workspace_bytes < qg_sample_tree_workspace_bytes(n_amps)) return fail(QG_E_INVALID_ARG, "workspace too small");
    const int64_t need = mode == 1 ? n_amps : std::min<int64_t>(shots, n_amps);
    if (capacity < need || (mode == 0 && !out_index_dev))
        return fail(QG_E_INVALID_ARG, "output capacity " + std::to_string(capacity) + " < " + std::to_string(need));
    cudaStream_t st = (cudaStream_t)stream;
    int64_t* nu = const_cast<int64_t*>(qg::tree_nunique_ptr(workspace, n_amps));
    QG_CUDA(qg::tree_draw(state, n_amps, dtype, workspace, shots, seed, tag, mode, index_base, out_index_dev,
                          out_count_dev, mode == 0 ? nu : nullptr, st),
            "tree draw");
    if (n_out_dev && mode == 0)
        QG_CUDA(cudaMemcpyAsync(n_out_dev, nu, 8, cudaMemcpyDeviceToDevice, st), "nunique copy");
    if (n_out_host) {
        if (mode == 0) {
            QG_CUDA(cudaMemcpyAsync(n_out_host, nu, 8, cudaMemcpyDeviceToHost, st), "nunique copy");
            QG_CUDA(cudaStreamSynchronize(st), "tree sync");
        } else {
            *n_out_host = n_amps;
        }
    }
    return QG_OK;
}

int qg_split_shots(const double* masses_host, int32_t n_parts, int64_t shots, uint64_t seed, void* workspace,
                   int64_t workspace_bytes, int64_t* counts_host, void* stream) {
    DeviceGuard dg_(workspace);
    if (!masses_host || !counts_host || !workspace || n_parts < 1 || n_parts > 64 || (n_parts & (n_parts - 1)) ||
        workspace_bytes < 1024 || shots < 0 || shots >= (1ll << 53))
        return fail(QG_E_INVALID_ARG, "bad split arguments");
    QG_CUDA(qg::tree_split_parts(masses_host, n_parts, shots, seed, workspace, counts_host, (cudaStream_t)stream),
            "split shots");
    return QG_OK;
}

int qg_binomial_test(double n, double p, uint64_t seed, int64_t count, int64_t* out_dev, void* stream) {
    DeviceGuard dg_(out_dev);
    if (!out_dev || count < 1 || !(n >= 0) || n >= 9007199254740992.0 || !(p >= 0 && p <= 1))
        return fail(QG_E_INVALID_ARG, "bad binomial test arguments");
    QG_CUDA(qg::binomial_test(n, p, seed, count, out_dev, (cudaStream_t)stream), "binomial test");
    return QG_OK;
}

}  // extern "C"
