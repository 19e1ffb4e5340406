// libtp C ABI entry points (include/tp.h): host-side argument validation and launches.
#include <cmath>
#include <cstring>
#include <new>

#include "tp_internal.cuh"

namespace {

bool freq_ok(const float* f, int32_t F) {
    if (!f || F < 1 || F > tp::kMaxF) return false;
    for (int u = 0; u < F; ++u) {
        if (!std::isfinite(f[u]) || !(f[u] > 0.f)) return false;
        if (u > 0 && !(f[u] > f[u - 1])) return false;
    }
    return true;
}

bool tbt_ok(float t) { return t >= 0x1p-17f && t <= 16.0f; }

bool H_ok(int32_t H) { return H >= 1 && H <= tp::kMaxH; }

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Makes the context's device current for one call (the launch helpers read per-device attributes
// of the current device) and restores the caller's on return.
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace

struct tp_ctx {
    int device;
    int32_t n_inst_max, n_req_max, H, F_max;
    int32_t *B, *KV, *n, *n_adm, *level;
    float* ips;
    void* work;
    size_t work_bytes;
    int k2_mode;
    int search;                   // TP_SEARCH_EXHAUSTIVE / TP_SEARCH_BINARY (K3 order)
    const tp_gbdt* cells_model;   // the model the workspace was sized for (cell mode), or null
    // admission control (tp_ctx_enable_admission): virtual prefix instances
    int32_t qc;
    tp_inst* vinst;
    int32_t *vforce, *vB, *vKV, *vn, *vnadm, *adm_final;
    uint32_t *vstatus, *lost;
    uint2* vres;
    void* vwork;
    size_t vwork_bytes;
    void* stage;     // tp_decide_host's device copy of the inputs: [inst | req | t_dead]
};

extern "C" {

const char* tp_strerror(int code) {
    switch (code) {
        case TP_OK: return "ok";
        case TP_EINVAL: return "invalid argument";
        case TP_ENOMEM: return "out of memory";
        case TP_ECUDA: return "CUDA error";
        case TP_EFORMAT: return "malformed or unsupported model blob";
        case TP_ENOTIMPL: return "not implemented";
        default: return "unknown error";
    }
}

int tp_abi_version(void) { return TP_ABI_VERSION; }

int tp_project(const tp_inst* inst, int32_t n_inst, const tp_req* req, int32_t n_req, int32_t H, int32_t* B,
               int32_t* KV, int32_t* n, int32_t* n_adm, uint32_t* status, void* stream) {
    if (n_inst < 0 || n_req < 0 || !H_ok(H)) return TP_EINVAL;
    if (n_inst > 0 && (!inst || !B || !KV || !n || !n_adm || !status || (n_req > 0 && !req))) return TP_EINVAL;
    return tp::launch_project(inst, n_inst, req, n_req, H, B, KV, n, n_adm, status, S(stream));
}

int tp_predict_ips(const tp_gbdt* m, const tp_inst* inst, int32_t n_inst, const int32_t* B, const int32_t* KV,
                   const int32_t* n, int32_t H, const float* freq_mhz, int32_t F, float* ips, uint32_t* status,
                   void* stream) {
    if (!m || n_inst < 0 || !H_ok(H) || !freq_ok(freq_mhz, F)) return TP_EINVAL;
    if (n_inst > 0 && (!inst || !B || !KV || !n || !ips || !status)) return TP_EINVAL;
    tp::K2Params p;
    std::memset(&p, 0, sizeof(p));
    p.words = m->m.d_words;
    p.cuts = m->m.d_cuts;
    for (int f = 0; f < 5; ++f) p.cut_off[f] = m->m.cut_off[f];
    p.rtab = m->m.d_rtab;
    for (int w = 0; w < 2; ++w) {
        p.rtab_off[w] = m->m.rtab_off[w];
        p.rtab_len[w] = m->m.rtab_len[w];
    }
    p.n_trees = m->m.n_trees;
    p.depth = m->m.depth;
    p.base = m->m.base;
    p.inst = inst;
    p.B = B;
    p.KV = KV;
    p.n = n;
    p.status = status;
    p.ips = ips;
    p.n_inst = n_inst;
    p.H = H;
    p.F = F;
    p.skip = TP_ST_BAD_INPUT | TP_ST_EMPTY | TP_ST_BYPASS_LOST;
    for (int u = 0; u < F; ++u) p.freq[u] = freq_mhz[u];
    return tp::launch_gbdt(p, false, S(stream));
}

size_t tp_predict_ips_workspace_size(const tp_gbdt* m, int32_t n_inst, int32_t H, int32_t F) {
    if (n_inst < 0 || !H_ok(H) || F < 1 || F > tp::kMaxF) return 0;
    return tp::runs_workspace_bytes(m ? tp::model_cells(m->m) : 0, n_inst, H, F);
}

static int predict_runs(const tp_gbdt* m, const tp_inst* inst, int32_t n_inst, const int32_t* B, const int32_t* KV,
                        const int32_t* n, int32_t H, const float* freq_mhz, int32_t F, float* ips, uint32_t* status,
                        void* workspace, size_t workspace_bytes, void* stream, uint32_t skip);

int tp_predict_ips_runs(const tp_gbdt* m, const tp_inst* inst, int32_t n_inst, const int32_t* B, const int32_t* KV,
                        const int32_t* n, int32_t H, const float* freq_mhz, int32_t F, float* ips, uint32_t* status,
                        void* workspace, size_t workspace_bytes, void* stream) {
    return predict_runs(m, inst, n_inst, B, KV, n, H, freq_mhz, F, ips, status, workspace, workspace_bytes, stream,
                        TP_ST_BAD_INPUT | TP_ST_EMPTY | TP_ST_BYPASS_LOST);
}

static int predict_runs(const tp_gbdt* m, const tp_inst* inst, int32_t n_inst, const int32_t* B, const int32_t* KV,
                        const int32_t* n, int32_t H, const float* freq_mhz, int32_t F, float* ips, uint32_t* status,
                        void* workspace, size_t workspace_bytes, void* stream, uint32_t skip) {
    if (!m || n_inst < 0 || !H_ok(H) || !freq_ok(freq_mhz, F)) return TP_EINVAL;
    if (n_inst > 0 && (!inst || !B || !KV || !n || !status || !workspace)) return TP_EINVAL;
    const int64_t cells = tp::model_cells(m->m);
    const bool use_cells = cells <= tp::kMaxCells && workspace_bytes >= tp::runs_workspace_bytes(cells, n_inst, H, F);
    if (n_inst > 0 && !ips && !use_cells) return TP_EINVAL;   // ips may be NULL only in cell mode
    if (n_inst > 0 && workspace_bytes < tp::runs_workspace_bytes(0, n_inst, H, F)) return TP_EINVAL;
    tp::K2Params p;
    std::memset(&p, 0, sizeof(p));
    p.words = m->m.d_words;
    p.cuts = m->m.d_cuts;
    for (int f = 0; f < 5; ++f) p.cut_off[f] = m->m.cut_off[f];
    p.rtab = m->m.d_rtab;
    for (int w = 0; w < 2; ++w) {
        p.rtab_off[w] = m->m.rtab_off[w];
        p.rtab_len[w] = m->m.rtab_len[w];
    }
    p.n_trees = m->m.n_trees;
    p.depth = m->m.depth;
    p.base = m->m.base;
    p.inst = inst;
    p.B = B;
    p.KV = KV;
    p.n = n;
    p.status = status;
    p.ips = ips;
    p.n_inst = n_inst;
    p.H = H;
    p.F = F;
    p.skip = skip;
    for (int u = 0; u < F; ++u) p.freq[u] = freq_mhz[u];
    if (n_inst > 0) tp::runs_workspace_carve(workspace, use_cells ? cells : 0, n_inst, H, F, p);
    return tp::launch_gbdt(p, true, S(stream));
}

int tp_runs_total(const void* workspace, int32_t n_inst, int32_t H, int64_t* total) {
    if (!workspace || !total || n_inst < 0 || !H_ok(H)) return TP_EINVAL;
    *total = 0;
    if (n_inst == 0) return TP_OK;
    tp::K2Params p;
    std::memset(&p, 0, sizeof(p));
    tp::runs_workspace_carve(const_cast<void*>(workspace), 0, n_inst, H, 1, p);
    int32_t* h = new (std::nothrow) int32_t[n_inst];
    if (!h) return TP_ENOMEM;
    const bool ok = cudaMemcpy(h, p.run_h, (size_t)n_inst * 4, cudaMemcpyDeviceToHost) == cudaSuccess;
    for (int32_t i = 0; ok && i < n_inst; ++i) *total += h[i];
    delete[] h;
    return ok ? TP_OK : TP_ECUDA;
}

int tp_cells_total(const tp_gbdt* m, const void* workspace, int32_t n_inst, int32_t H, int32_t F, int64_t* total) {
    if (!m || !workspace || !total || n_inst < 0 || !H_ok(H) || F < 1 || F > tp::kMaxF) return TP_EINVAL;
    *total = 0;
    tp::K2Params p;
    std::memset(&p, 0, sizeof(p));
    tp::runs_workspace_carve(const_cast<void*>(workspace), tp::model_cells(m->m), n_inst, H, F, p);
    if (!p.cell_count || n_inst == 0) return TP_OK;
    int32_t c = 0;
    if (cudaMemcpy(&c, p.cell_count, 4, cudaMemcpyDeviceToHost) != cudaSuccess) return TP_ECUDA;
    *total = (int64_t)c + 1;   // stored as count - 1
    return TP_OK;
}

int tp_compact_stats(const tp_gbdt* m, const void* workspace, size_t workspace_bytes, int32_t n_inst, int32_t H,
                     int32_t F, int64_t* out) {
    if (!m || !out || n_inst < 0 || !H_ok(H) || F < 1 || F > tp::kMaxF) return TP_EINVAL;
    out[0] = out[1] = out[2] = 0;
    if (n_inst == 0) return TP_OK;
    const int64_t cells = tp::model_cells(m->m);
    if (!workspace || cells > tp::kMaxCells || workspace_bytes < tp::runs_workspace_bytes(cells, n_inst, H, F))
        return TP_EINVAL;
    tp::K2Params p;
    std::memset(&p, 0, sizeof(p));
    tp::runs_workspace_carve(const_cast<void*>(workspace), cells, n_inst, H, F, p);
    int32_t* h = new (std::nothrow) int32_t[2 * (size_t)n_inst];
    if (!h) return TP_ENOMEM;
    int32_t c = -1;
    const bool ok = cudaMemcpy(h, p.run_h, (size_t)n_inst * 4, cudaMemcpyDeviceToHost) == cudaSuccess &&
                    cudaMemcpy(h + n_inst, p.end_n, (size_t)n_inst * 4, cudaMemcpyDeviceToHost) == cudaSuccess &&
                    cudaMemcpy(&c, p.cell_count, 4, cudaMemcpyDeviceToHost) == cudaSuccess;
    for (int32_t i = 0; ok && i < n_inst; ++i) {
        out[0] += h[i];
        out[1] += h[n_inst + i];
    }
    out[2] = (int64_t)c + 1;
    delete[] h;
    return ok ? TP_OK : TP_ECUDA;
}

int tp_select_freq(const tp_inst* inst, int32_t n_inst, const tp_req* req, int32_t n_req, const double* t_dead,
                   const int32_t* n, const int32_t* n_adm, const float* ips, int32_t H, int32_t F, float tbt_slo,
                   int32_t* level, uint32_t* status, int64_t* tr_ticks, void* stream) {
    if (n_inst < 0 || n_req < 0 || !H_ok(H) || F < 1 || F > tp::kMaxF || !tbt_ok(tbt_slo)) return TP_EINVAL;
    if (n_inst > 0 && (!inst || !n || !n_adm || !ips || !level || !status || (n_req > 0 && (!req || !t_dead))))
        return TP_EINVAL;
    const int64_t tbt_ticks = (int64_t)((double)tbt_slo * 0x1p40);   // exact: tbt_slo >= 2^-17
    return tp::launch_select(inst, n_inst, req, n_req, t_dead, n, n_adm, ips, H, F, tbt_ticks, level, status,
                             tr_ticks, nullptr, TP_SEARCH_EXHAUSTIVE, S(stream));
}

static int select_ws(const tp_gbdt* m, const void* workspace, const tp_inst* inst, int32_t n_inst, const tp_req* req,
                     int32_t n_req, const double* t_dead, const int32_t* n, const int32_t* n_adm, int32_t H, int32_t F,
                     float tbt_slo, int32_t* level, uint32_t* status, int64_t* tr_ticks, int search, void* stream) {
    if (!m || n_inst < 0 || n_req < 0 || !H_ok(H) || H > tp::kMaxHRunsSelect || F < 1 || F > tp::kMaxF ||
        !tbt_ok(tbt_slo))
        return TP_EINVAL;
    if (n_inst > 0 && (!workspace || !inst || !n || !n_adm || !level || !status || (n_req > 0 && (!req || !t_dead))))
        return TP_EINVAL;
    tp::K2Params p;
    std::memset(&p, 0, sizeof(p));
    tp::runs_workspace_carve(const_cast<void*>(workspace), tp::model_cells(m->m), n_inst, H, F, p);
    if (n_inst > 0 && !p.cell_tab) return TP_EINVAL;   // the model has no cell mode
    const int64_t tbt_ticks = (int64_t)((double)tbt_slo * 0x1p40);
    return tp::launch_select(inst, n_inst, req, n_req, t_dead, n, n_adm, nullptr, H, F, tbt_ticks, level, status,
                             tr_ticks, &p, search, S(stream));
}

int tp_select_freq_ws(const tp_gbdt* m, const void* workspace, const tp_inst* inst, int32_t n_inst, const tp_req* req,
                      int32_t n_req, const double* t_dead, const int32_t* n, const int32_t* n_adm, int32_t H, int32_t F,
                      float tbt_slo, int32_t* level, uint32_t* status, int64_t* tr_ticks, void* stream) {
    return select_ws(m, workspace, inst, n_inst, req, n_req, t_dead, n, n_adm, H, F, tbt_slo, level, status, tr_ticks,
                     TP_SEARCH_EXHAUSTIVE, stream);
}

int tp_select_freq_binary(const tp_gbdt* m, const void* workspace, const tp_inst* inst, int32_t n_inst,
                          const tp_req* req, int32_t n_req, const double* t_dead, const int32_t* n, const int32_t* n_adm,
                          int32_t H, int32_t F, float tbt_slo, int32_t* level, uint32_t* status, void* stream) {
    return select_ws(m, workspace, inst, n_inst, req, n_req, t_dead, n, n_adm, H, F, tbt_slo, level, status, nullptr,
                     TP_SEARCH_BINARY, stream);
}

static void fill_model(const tp_gbdt* m, tp::K2Params& p) {
    p.words = m->m.d_words;
    p.cuts = m->m.d_cuts;
    for (int f = 0; f < 5; ++f) p.cut_off[f] = m->m.cut_off[f];
    p.rtab = m->m.d_rtab;
    for (int w = 0; w < 2; ++w) {
        p.rtab_off[w] = m->m.rtab_off[w];
        p.rtab_len[w] = m->m.rtab_len[w];
    }
    p.n_trees = m->m.n_trees;
    p.depth = m->m.depth;
    p.base = m->m.base;
    p.tick_shift = m->m.tick_shift;
}

static bool compact_ws_ok(const tp_gbdt* m, size_t bytes, int32_t n_inst, int32_t H, int32_t F) {
    const int64_t cells = tp::model_cells(m->m);
    return cells <= tp::kMaxCells && bytes >= tp::runs_workspace_bytes(cells, n_inst, H, F);
}

int tp_project_compact(const tp_gbdt* m, void* workspace, size_t workspace_bytes, const tp_inst* inst,
                       int32_t n_inst, const tp_req* req, int32_t n_req, const double* t_dead, int32_t H, int32_t* B,
                       int32_t* KV, int32_t bkv_rows, int32_t* n, int32_t* n_adm, uint32_t* status, void* stream) {
    if (!m || n_inst < 0 || n_req < 0 || !H_ok(H) || (bkv_rows != 0 && bkv_rows != 1) || (!B) != (!KV))
        return TP_EINVAL;
    if (n_inst == 0) return TP_OK;
    if (!workspace || !inst || !n || !n_adm || !status || (n_req > 0 && (!req || !t_dead)) ||
        !compact_ws_ok(m, workspace_bytes, n_inst, H, 1))
        return TP_EINVAL;
    tp::K2Params p;
    std::memset(&p, 0, sizeof(p));
    fill_model(m, p);
    tp::runs_workspace_carve(workspace, tp::model_cells(m->m), n_inst, H, 1, p);
    return tp::launch_project_compact(p, inst, n_inst, req, n_req, t_dead, H, B, KV, bkv_rows, n, n_adm, status,
                                      TP_ST_BAD_INPUT | TP_ST_EMPTY | TP_ST_BYPASS_LOST, S(stream));
}

int tp_predict_cells(const tp_gbdt* m, void* workspace, size_t workspace_bytes, int32_t n_inst, int32_t H,
                     const float* freq_mhz, int32_t F, void* stream) {
    if (!m || n_inst < 0 || !H_ok(H) || !freq_ok(freq_mhz, F)) return TP_EINVAL;
    if (n_inst == 0) return TP_OK;
    if (!workspace || !compact_ws_ok(m, workspace_bytes, n_inst, H, F)) return TP_EINVAL;
    tp::K2Params p;
    std::memset(&p, 0, sizeof(p));
    fill_model(m, p);
    p.n_inst = n_inst;
    p.H = H;
    p.F = F;
    p.skip = TP_ST_BAD_INPUT | TP_ST_EMPTY | TP_ST_BYPASS_LOST;
    p.runs_ready = 1;
    for (int u = 0; u < F; ++u) p.freq[u] = freq_mhz[u];
    tp::runs_workspace_carve(workspace, tp::model_cells(m->m), n_inst, H, F, p);
    return tp::launch_gbdt(p, true, S(stream));
}

int tp_select_freq_compact(const tp_gbdt* m, const void* workspace, size_t workspace_bytes, int32_t n_inst,
                           const int32_t* n, int32_t H, int32_t F, float tbt_slo, int32_t search, int32_t* level,
                           uint32_t* status, void* stream) {
    if (!m || n_inst < 0 || !H_ok(H) || F < 1 || F > tp::kMaxF || !tbt_ok(tbt_slo) ||
        (search != TP_SEARCH_EXHAUSTIVE && search != TP_SEARCH_BINARY))
        return TP_EINVAL;
    if (n_inst == 0) return TP_OK;
    if (!workspace || !n || !level || !status || !compact_ws_ok(m, workspace_bytes, n_inst, H, F)) return TP_EINVAL;
    tp::K2Params p;
    std::memset(&p, 0, sizeof(p));
    tp::runs_workspace_carve(const_cast<void*>(workspace), tp::model_cells(m->m), n_inst, H, F, p);
    p.tick_shift = m->m.tick_shift;
    const int64_t tbt_ticks = (int64_t)((double)tbt_slo * 0x1p40);   // exact: tbt_slo >= 2^-17
    return tp::launch_select_compact(p, n_inst, n, H, F, tbt_ticks, search,
                                     TP_ST_BAD_INPUT | TP_ST_EMPTY | TP_ST_BYPASS_LOST, level, status, S(stream));
}

int tp_replay_advance(const tp_gbdt* m, tp_inst* inst, int32_t n_inst, const tp_req* req, const double* t_dead,
                      tp_req* req_out, double* t_dead_out, int32_t slot_cap, int32_t H, const int32_t* B,
                      const int32_t* KV, const int32_t* n, const int32_t* n_adm, const uint32_t* status,
                      const int32_t* level, const float* freq_mhz, int32_t F, const double* arr_t,
                      const tp_req* arr_req, const double* arr_dead, const int64_t* arr_off, int64_t* arr_next,
                      uint64_t* stats, const uint32_t* adm_lost, void* stream) {
    if (!m || n_inst < 0 || slot_cap < 1 || !H_ok(H) || !freq_ok(freq_mhz, F)) return TP_EINVAL;
    if (n_inst > 0 && (!inst || !req || !t_dead || !req_out || !t_dead_out || !B || !KV || !n || !n_adm || !status ||
                       !level || !arr_t || !arr_req || !arr_dead || !arr_off || !arr_next || !stats))
        return TP_EINVAL;
    return tp::launch_replay_advance(m->m, inst, n_inst, req, t_dead, req_out, t_dead_out, slot_cap, H, B, KV, n,
                                     n_adm, status, level, freq_mhz, F, arr_t, arr_req, arr_dead, arr_off, arr_next,
                                     reinterpret_cast<unsigned long long*>(stats), adm_lost, S(stream));
}

int tp_ctx_create(int device, const tp_gbdt* model, int32_t n_inst_max, int32_t n_req_max, int32_t H, int32_t F_max,
                  tp_ctx** out) {
    if (!out || n_inst_max < 0 || n_req_max < 0 || !H_ok(H) || F_max < 1 || F_max > tp::kMaxF) return TP_EINVAL;
    *out = nullptr;
    tp_ctx* c = new (std::nothrow) tp_ctx();
    if (!c) return TP_ENOMEM;
    std::memset(c, 0, sizeof(*c));
    c->device = device;
    c->n_inst_max = n_inst_max;
    c->n_req_max = n_req_max;
    c->H = H;
    c->F_max = F_max;
    c->cells_model = (model && tp::model_cells(model->m) <= tp::kMaxCells) ? model : nullptr;
    c->k2_mode = c->cells_model ? TP_K2_COMPACT : TP_K2_RUNS;
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) {
        delete c;
        return TP_ECUDA;
    }
    const size_t I = (size_t)(n_inst_max > 0 ? n_inst_max : 1), R = (size_t)(n_req_max > 0 ? n_req_max : 1);
    bool ok = cudaMalloc(&c->B, I * H * 4) == cudaSuccess && cudaMalloc(&c->KV, I * H * 4) == cudaSuccess &&
              cudaMalloc(&c->n, I * 4) == cudaSuccess && cudaMalloc(&c->n_adm, I * 4) == cudaSuccess &&
              cudaMalloc(&c->level, I * 8) == cudaSuccess &&   // [level | status] of the last call, contiguous
              // the ips grid only for the paths that write it (allocated on demand by set_k2_mode)
              (c->cells_model || cudaMalloc(&c->ips, I * F_max * H * 4) == cudaSuccess) &&
              cudaMalloc(&c->work, c->work_bytes = tp::runs_workspace_bytes(model ? tp::model_cells(model->m) : 0,
                                                                            (int32_t)I, H, F_max)) == cudaSuccess &&
              // host-input staging [inst | req | t_dead], carved per call (tp_decide_host)
              cudaMalloc(&c->stage, I * sizeof(tp_inst) + R * (sizeof(tp_req) + sizeof(double))) == cudaSuccess;
    cudaSetDevice(prev);
    if (!ok) {
        tp_ctx_free(c);
        return TP_ENOMEM;
    }
    *out = c;
    return TP_OK;
}

int tp_ctx_free(tp_ctx* c) {
    if (!c) return TP_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    void* ptrs[] = {c->B,     c->KV,    c->n,      c->n_adm,     c->level, c->ips,   c->work,
                    c->stage, c->vinst,     c->vforce, c->vB,   c->vKV,   c->vn,
                    c->vnadm, c->adm_final, c->vstatus, c->lost, c->vres,  c->vwork};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    cudaSetDevice(prev);
    delete c;
    return TP_OK;
}

int tp_ctx_enable_admission(tp_ctx* c, int32_t q_max) {
    if (!c || q_max < 1 || q_max > 32 || !c->cells_model || c->H > tp::kMaxHRunsSelect) return TP_EINVAL;
    if (c->qc) return c->qc == q_max ? TP_OK : TP_EINVAL;
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(c->device) != cudaSuccess) return TP_ECUDA;
    const size_t I = (size_t)(c->n_inst_max > 0 ? c->n_inst_max : 1), V = I * q_max, H = c->H;
    c->vwork_bytes = tp::runs_workspace_bytes(tp::model_cells(c->cells_model->m), (int32_t)V, c->H, 1);
    const bool ok = cudaMalloc(&c->vinst, V * sizeof(tp_inst)) == cudaSuccess &&
                    cudaMalloc(&c->vforce, V * 4) == cudaSuccess && cudaMalloc(&c->vB, V * H * 4) == cudaSuccess &&
                    cudaMalloc(&c->vKV, V * H * 4) == cudaSuccess && cudaMalloc(&c->vn, V * 4) == cudaSuccess &&
                    cudaMalloc(&c->vnadm, V * 4) == cudaSuccess && cudaMalloc(&c->vstatus, V * 4) == cudaSuccess &&
                    cudaMalloc(&c->vres, V * sizeof(uint2)) == cudaSuccess &&
                    cudaMalloc(&c->adm_final, I * 4) == cudaSuccess && cudaMalloc(&c->lost, I * 4) == cudaSuccess &&
                    cudaMalloc(&c->vwork, c->vwork_bytes) == cudaSuccess;
    cudaSetDevice(prev);
    if (!ok) return TP_ENOMEM;
    c->qc = q_max;
    return TP_OK;
}

int tp_decide_admit(tp_ctx* c, const tp_gbdt* m, const tp_inst* inst, int32_t n_inst, const tp_req* req,
                    int32_t n_req, const double* t_dead, const float* freq_mhz, int32_t F, float tbt_slo,
                    int32_t* level, uint32_t* status, int32_t* n_adm_out, uint32_t* adm_lost_out, void* stream) {
    if (!c) return TP_EINVAL;
    DeviceGuard dg(c->device);
    if (!dg.ok) return TP_ECUDA;
    if (!c || !m || !c->qc || m != c->cells_model || n_inst < 0 || n_inst > c->n_inst_max || F > c->F_max ||
        !freq_ok(freq_mhz, F) || !tbt_ok(tbt_slo))
        return TP_EINVAL;
    if (n_inst > 0 && (!inst || !level || !status || (n_req > 0 && (!req || !t_dead)))) return TP_EINVAL;
    if (n_inst == 0) return TP_OK;
    cudaStream_t s = S(stream);
    const int32_t V = n_inst * c->qc, H = c->H;
    const int64_t tbt_ticks = (int64_t)((double)tbt_slo * 0x1p40);
    // 1. check 1 + batch cap (K1 gate): the longest admissible prefix
    int rc = tp::launch_project(inst, n_inst, req, n_req, H, c->B, c->KV, c->n, c->n_adm, status, s);
    // 2. every prefix as a virtual instance, its candidates forced in
    if (!rc) rc = tp::launch_admit_expand(inst, n_inst, c->qc, c->n_adm, status, c->vinst, c->vforce, s);
    // 3. M at the maximum frequency on every prefix state (cell mode, LUT only)
    // (a lost running request does not exempt the prefix from the checks: only BAD / EMPTY are skipped)
    const bool compact = c->k2_mode == TP_K2_COMPACT;
    tp::K2Params w;
    std::memset(&w, 0, sizeof(w));
    fill_model(m, w);
    tp::runs_workspace_carve(c->vwork, tp::model_cells(m->m), V, H, 1, w);
    if (compact) {
        // K1c builds the prefix states' runs and cells directly; K2 evaluates the cells at f_max
        if (!rc) rc = tp::launch_project_compact(w, c->vinst, V, req, n_req, t_dead, H, nullptr, nullptr, 0, c->vn,
                                                 c->vnadm, c->vstatus, TP_ST_BAD_INPUT | TP_ST_EMPTY, s, c->vforce,
                                                 nullptr);
        tp::K2Params k = w;
        k.n_inst = V;
        k.H = H;
        k.F = 1;
        k.freq[0] = freq_mhz[F - 1];
        k.skip = TP_ST_BAD_INPUT | TP_ST_EMPTY;
        k.runs_ready = 1;
        if (!rc) rc = tp::launch_gbdt(k, true, s);
    } else {
        if (!rc) rc = tp::launch_project(c->vinst, V, req, n_req, H, c->vB, c->vKV, c->vn, c->vnadm, c->vstatus, s,
                                         c->vforce, nullptr);
        if (!rc) rc = predict_runs(m, c->vinst, V, c->vB, c->vKV, c->vn, H, freq_mhz + (F - 1), 1, nullptr,
                                   c->vstatus, c->vwork, c->vwork_bytes, stream, TP_ST_BAD_INPUT | TP_ST_EMPTY);
    }
    // 4. checks 2-3 per prefix, 5. FIFO resolution with lost marks
    if (!rc) rc = tp::launch_admit_checks(c->vinst, V, req, t_dead, c->vn, c->vstatus, w, H, tbt_ticks, c->vres, s);
    if (!rc) rc = tp::launch_admit_resolve(n_inst, c->qc, inst, status, c->n_adm, c->vres, c->adm_final, c->lost, s);
    // 6. the throttle on the admitted state (lost marks applied -> bypass)
    if (compact) {
        tp::K2Params w2;
        std::memset(&w2, 0, sizeof(w2));
        fill_model(m, w2);
        tp::runs_workspace_carve(c->work, tp::model_cells(m->m), n_inst, H, 1, w2);
        if (!rc) rc = tp::launch_project_compact(w2, inst, n_inst, req, n_req, t_dead, H, c->B, c->KV, 0, c->n,
                                                 c->n_adm, status, TP_ST_BAD_INPUT | TP_ST_EMPTY | TP_ST_BYPASS_LOST,
                                                 s, c->adm_final, c->lost);
        if (!rc) rc = tp_predict_cells(m, c->work, c->work_bytes, n_inst, H, freq_mhz, F, stream);
        if (!rc) rc = tp_select_freq_compact(m, c->work, c->work_bytes, n_inst, c->n, H, F, tbt_slo, c->search, level,
                                             status, stream);
    } else {
        if (!rc) rc = tp::launch_project(inst, n_inst, req, n_req, H, c->B, c->KV, c->n, c->n_adm, status, s,
                                         c->adm_final, c->lost);
        if (!rc) rc = tp_predict_ips_runs(m, inst, n_inst, c->B, c->KV, c->n, H, freq_mhz, F, nullptr, status,
                                          c->work, c->work_bytes, stream);
        if (!rc) rc = select_ws(m, c->work, inst, n_inst, req, n_req, t_dead, c->n, c->n_adm, H, F, tbt_slo, level,
                                status, nullptr, c->search, stream);
    }
    if (!rc && n_adm_out && cudaMemcpyAsync(n_adm_out, c->n_adm, (size_t)n_inst * 4, cudaMemcpyDeviceToDevice, s))
        rc = TP_ECUDA;
    if (!rc && adm_lost_out &&
        cudaMemcpyAsync(adm_lost_out, c->lost, (size_t)n_inst * 4, cudaMemcpyDeviceToDevice, s))
        rc = TP_ECUDA;
    return rc;
}

int tp_ctx_set_k2_mode(tp_ctx* c, int mode) {
    if (!c || (mode != TP_K2_DIRECT && mode != TP_K2_RUNS && mode != TP_K2_COMPACT)) return TP_EINVAL;
    if (mode != TP_K2_COMPACT && !c->ips) {   // direct / run / cell modes may write the ips grid
        const size_t I = (size_t)(c->n_inst_max > 0 ? c->n_inst_max : 1);
        int prev = 0;
        cudaGetDevice(&prev);
        if (cudaSetDevice(c->device) != cudaSuccess) return TP_ECUDA;
        const bool ok = cudaMalloc(&c->ips, I * c->F_max * c->H * 4) == cudaSuccess;
        cudaSetDevice(prev);
        if (!ok) {
            c->ips = nullptr;
            return TP_ENOMEM;
        }
    }
    c->k2_mode = mode;
    return TP_OK;
}

int tp_ctx_set_search(tp_ctx* c, int search) {
    if (!c || (search != TP_SEARCH_EXHAUSTIVE && search != TP_SEARCH_BINARY)) return TP_EINVAL;
    c->search = search;
    return TP_OK;
}

int tp_ctx_buffers(tp_ctx* c, int32_t** B, int32_t** KV, int32_t** n, int32_t** n_adm, float** ips) {
    if (!c) return TP_EINVAL;
    if (B) *B = c->B;
    if (KV) *KV = c->KV;
    if (n) *n = c->n;
    if (n_adm) *n_adm = c->n_adm;
    if (ips) *ips = c->ips;
    return TP_OK;
}

int tp_decide(tp_ctx* c, const tp_gbdt* m, const tp_inst* inst, int32_t n_inst, const tp_req* req, int32_t n_req,
              const double* t_dead, const float* freq_mhz, int32_t F, float tbt_slo, int32_t* level,
              uint32_t* status, void* stream) {
    if (!c) return TP_EINVAL;
    DeviceGuard dg(c->device);
    if (!dg.ok) return TP_ECUDA;
    if (!c || !m || n_inst < 0 || n_inst > c->n_inst_max || F > c->F_max || !freq_ok(freq_mhz, F) ||
        !tbt_ok(tbt_slo))
        return TP_EINVAL;
    const bool cells = c->k2_mode != TP_K2_DIRECT && c->cells_model == m && m != nullptr;
    if (c->k2_mode == TP_K2_COMPACT) {
        // K1c -> K2 (cells) -> K3c: B/KV stay on chip (only m = 1 is written, for tp_replay_advance)
        if (!cells) return TP_ENOTIMPL;
        int rc = tp_project_compact(m, c->work, c->work_bytes, inst, n_inst, req, n_req, t_dead, c->H, c->B, c->KV,
                                    0, c->n, c->n_adm, status, stream);
        if (!rc) rc = tp_predict_cells(m, c->work, c->work_bytes, n_inst, c->H, freq_mhz, F, stream);
        if (!rc) rc = tp_select_freq_compact(m, c->work, c->work_bytes, n_inst, c->n, c->H, F, tbt_slo, c->search,
                                             level, status, stream);
        return rc;
    }
    // cell mode (ctx created with the model): K2 leaves the IPS values in the LUT and K3 reads them
    // through the runs -- the ips grid is never materialised
    const bool fused = c->k2_mode == TP_K2_RUNS && cells && c->H <= tp::kMaxHRunsSelect;
    if (c->search == TP_SEARCH_BINARY && !fused) return TP_ENOTIMPL;   // binary search reads the cell LUT
    int rc = tp_project(inst, n_inst, req, n_req, c->H, c->B, c->KV, c->n, c->n_adm, status, stream);
    if (rc) return rc;
    if (c->k2_mode == TP_K2_RUNS)
        rc = tp_predict_ips_runs(m, inst, n_inst, c->B, c->KV, c->n, c->H, freq_mhz, F, fused ? nullptr : c->ips,
                                 status, c->work, c->work_bytes, stream);
    else
        rc = tp_predict_ips(m, inst, n_inst, c->B, c->KV, c->n, c->H, freq_mhz, F, c->ips, status, stream);
    if (rc) return rc;
    if (fused)
        return select_ws(m, c->work, inst, n_inst, req, n_req, t_dead, c->n, c->n_adm, c->H, F, tbt_slo, level,
                         status, nullptr, c->search, stream);
    return tp_select_freq(inst, n_inst, req, n_req, t_dead, c->n, c->n_adm, c->ips, c->H, F, tbt_slo, level, status,
                          nullptr, stream);
}

int tp_decide_host(tp_ctx* c, const tp_gbdt* m, const tp_inst* h_inst, int32_t n_inst, const tp_req* h_req,
                   int32_t n_req, const double* h_t_dead, const float* freq_mhz, int32_t F, float tbt_slo,
                   int32_t* h_level, uint32_t* h_status, void* stream) {
    if (!c) return TP_EINVAL;
    DeviceGuard dg(c->device);
    if (!dg.ok) return TP_ECUDA;
    if (!c || !m || n_inst < 0 || n_inst > c->n_inst_max || n_req < 0 || n_req > c->n_req_max) return TP_EINVAL;
    if (n_inst > 0 && (!h_inst || !h_level || !h_status || (n_req > 0 && (!h_req || !h_t_dead)))) return TP_EINVAL;
    if (!freq_ok(freq_mhz, F) || F > c->F_max || !tbt_ok(tbt_slo)) return TP_EINVAL;
    cudaStream_t s = S(stream);
    // device staging laid out like a packed host buffer [inst | req | t_dead] (offsets 16-byte /
    // 8-byte aligned for any counts); when the caller's buffers are packed that way, one copy
    char* base = static_cast<char*>(c->stage);
    const size_t bi = (size_t)n_inst * sizeof(tp_inst), br = (size_t)n_req * sizeof(tp_req),
                 bd = (size_t)n_req * sizeof(double);
    tp_inst* d_inst = reinterpret_cast<tp_inst*>(base);
    tp_req* d_req = reinterpret_cast<tp_req*>(base + bi);
    double* d_dead = reinterpret_cast<double*>(base + bi + br);
    const char* hi = reinterpret_cast<const char*>(h_inst);
    const bool packed = n_inst > 0 && n_req > 0 && reinterpret_cast<const char*>(h_req) == hi + bi &&
                        reinterpret_cast<const char*>(h_t_dead) == hi + bi + br;
    if (packed) {
        if (cudaMemcpyAsync(base, h_inst, bi + br + bd, cudaMemcpyHostToDevice, s)) return TP_ECUDA;
    } else if (cudaMemcpyAsync(d_inst, h_inst, bi, cudaMemcpyHostToDevice, s) ||
               (br && cudaMemcpyAsync(d_req, h_req, br, cudaMemcpyHostToDevice, s)) ||
               (bd && cudaMemcpyAsync(d_dead, h_t_dead, bd, cudaMemcpyHostToDevice, s))) {
        return TP_ECUDA;
    }
    int32_t* d_level = c->level;
    uint32_t* d_status = reinterpret_cast<uint32_t*>(c->level + n_inst);
    int rc = tp_decide(c, m, d_inst, n_inst, d_req, n_req, d_dead, freq_mhz, F, tbt_slo, d_level, d_status, stream);
    if (rc) return rc;
    if (reinterpret_cast<const char*>(h_status) == reinterpret_cast<const char*>(h_level) + (size_t)n_inst * 4) {
        if (cudaMemcpyAsync(h_level, d_level, (size_t)n_inst * 8, cudaMemcpyDeviceToHost, s)) return TP_ECUDA;
    } else if (cudaMemcpyAsync(h_level, d_level, (size_t)n_inst * 4, cudaMemcpyDeviceToHost, s) ||
               cudaMemcpyAsync(h_status, d_status, (size_t)n_inst * 4, cudaMemcpyDeviceToHost, s)) {
        return TP_ECUDA;
    }
    return TP_OK;
}

}  // extern "C"
