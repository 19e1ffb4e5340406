/*
 * tp.h -- C ABI of libtp: throttLL'eM's per-iteration GPU-frequency-selection hot path
 * (arXiv 2408.05235, "SLO-aware GPU Frequency Scaling for Energy Efficient LLM Inference
 * Serving"), implemented as hand-written sm_100a CUDA kernels.
 *
 * Citations: P:L = line L of the paper text; readings A-n of ambiguous passages are
 * listed in DESIGN.md §3.
 *
 * The path, per serving instance (one LLM engine with its Scoreboard):
 *   tp_project      K1  Eq. 1-2 projection of batch size B[m] and KV blocks KV[m] for the future
 *                       iterations m = 1..H (m = 1 is the iteration about to run, reading A-1),
 *                       with FIFO admission of queued requests by check 1 + batch cap.
 *   tp_predict_ips  K2  the GBDT performance model M(tp, B[m], KV[m], f) -> IPS on
 *                       the full (instance x frequency x iteration m <= n) grid.
 *   tp_select_freq  K3  T' = 1/IPS, T_R = cumulative sum (Eq. 3), TBT check
 *                        and Eq. 4 deadlines, lowest passing frequency.
 *
 * General conventions (all calls):
 *   - Pointers marked [dev] are device pointers, [host] host pointers; all are owned by the
 *     caller.  The library never frees caller memory; only tp_gbdt_load / tp_ctx_create allocate.
 *   - Kernels are enqueued on `stream` (a cudaStream_t; NULL = legacy default stream) and the
 *     call returns after enqueue.  No call allocates or synchronises except the two creators,
 *     tp_gbdt_free / tp_ctx_free, and tp_decide_host (which only enqueues copies on `stream`).
 *   - Host-detectable argument errors return TP_EINVAL and enqueue nothing: NULL pointers with
 *     n_inst > 0, n_inst < 0, H outside [1, 16384], F outside [1, 32], non-finite, non-positive
 *     or non-ascending frequencies, tbt_slo outside [2^-17, 16] s.
 *   - Device-detected errors in ONE instance's data never fail the batch: the instance gets
 *     status TP_ST_BAD_INPUT, level F-1, n = n_adm = 0 and zero curves.  Bad data is any of:
 *     N < 1, tp < 1, tp >= 2^24, n_run < 0, n_queue < 0, kv_cap < 0, max_batch < 0,
 *     req_begin < 0, req_begin + n_run + n_queue > n_req; any entry with a < 0, q < 1, r < 1,
 *     a >= 2^24, q >= 2^24, or l = r - a outside [1, H] (reading A-3; l <= 0 is a length
 *     overrun the caller fixes); a queued entry with a != 0; or a total footprint
 *     sum_e ceil((a_e + l_e - 1 + q_e) / N) >= 2^24 (keeps KV exact as an fp32 feature).
 *   - Launch failures return TP_ECUDA; malformed model blobs TP_EFORMAT.
 *   - Calls on different streams may run concurrently; a tp_gbdt handle is immutable and may be
 *     shared by any number of concurrent calls on its device.
 */
#ifndef TP_H
#define TP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TP_ABI_VERSION 1

/* ---- return codes ---- */
enum {
    TP_OK = 0,
    TP_EINVAL = -1,   /* bad argument, nothing enqueued */
    TP_ENOMEM = -2,   /* device / host allocation failed (creators only) */
    TP_ECUDA = -3,    /* a CUDA call or launch failed */
    TP_EFORMAT = -4,  /* malformed or unsupported model blob */
    TP_ENOTIMPL = -5
};

/* ---- per-instance status bits (uint32, OR-ed) ---- */
enum {
    TP_ST_EMPTY = 1,          /* n = 0: nothing scheduled; level 0 (reading A-15) */
    TP_ST_BYPASS_LOST = 2,    /* a "lost" request is scheduled -> max frequency */
    TP_ST_INFEASIBLE = 4,     /* no level meets the SLOs -> level F-1 (reading A-14) */
    TP_ST_KV_OVER = 8,        /* running requests alone exceed kv_cap somewhere */
    TP_ST_QUEUE_BLOCKED = 16, /* a queued request failed check 1 / batch cap; FIFO stop */
    TP_ST_IPS_CLAMPED = 32,   /* a model output was clamped to [2^-4, 2^17] (reading A-8) */
    TP_ST_BAD_INPUT = 64      /* invalid instance data (see conventions) */
};
/* level precedence: BAD_INPUT (F-1) > EMPTY (0) > BYPASS_LOST (F-1) > lowest passing level >
 * INFEASIBLE (F-1). */

#define TP_REQ_LOST 1u        /* tp_req.flags bit 0: request marked "lost" */

/* Instance header, 48 bytes, little-endian, 8-byte aligned.  One per serving instance. */
typedef struct tp_inst {
    int64_t k;          /* current iteration k (informational; requests carry a = k - s_i) */
    double t_cur;       /* current time t_cur in seconds (Eq. 4) */
    int32_t req_begin;  /* index of this instance's first request in the request array */
    int32_t n_run;      /* running (scheduled) requests, stored first */
    int32_t n_queue;    /* queued requests, stored next in FIFO order */
    int32_t N;          /* tokens per KV block ("compile time parameter"; reading A-4) */
    int32_t kv_cap;     /* KV-cache capacity in blocks (check 1) */
    int32_t max_batch;  /* engine batch-size cap (admission reading A-2) */
    int32_t tp;         /* engine size / tensor-parallel degree: model feature 0 */
    int32_t _pad;       /* must be ignored */
} tp_inst;

/* Scoreboard entry, 16 bytes.  Running entries: a = k - s_i >= 0 iterations since it
 * was scheduled; queued entries: a = 0 (virtual append at s = k).  q = |q_i| prompt
 * tokens, r = r^_i predicted generation length (already conservatively adjusted).
 * The entry completes at iteration s_i + r^_i, i.e. at l = r - a. */
typedef struct tp_req {
    int32_t a, q, r;
    uint32_t flags;     /* bit 0: TP_REQ_LOST */
} tp_req;

typedef struct tp_gbdt tp_gbdt;   /* opaque, immutable model on one device */

typedef struct tp_gbdt_info {
    int32_t n_trees;      /* T */
    int32_t depth;        /* D: trees are stored complete to this depth */
    int32_t n_cuts[4];    /* distinct thresholds per feature [tp, batch, kv, freq] */
    float base_score;
    int32_t tick_shift;   /* 8: every output is in (1, 512) IPS, T' kept as 32-bit (tick / 2^8) */
    int64_t device_bytes; /* bytes of device memory held by the handle */
    int64_t node_bytes;   /* bytes of the node arrays (T * 2^(D+1) * 4) */
} tp_gbdt_info;

/*
 * Model blob v1 (little-endian; host memory, caller keeps ownership):
 *   char magic[4] = "TPGB"; u32 version = 1; u32 n_features = 4 (order [tp, batch, kv_blocks,
 *   freq_mhz]); u32 n_trees; u32 max_depth (<= 12); f32 base_score;
 *   per tree: u32 n_nodes (1..8192) then n_nodes x {i32 feature (-1 = leaf), f32 threshold,
 *   i32 left, i32 right, f32 leaf_value}; node 0 is the root.
 * Semantics (XGBoost convention, reading A-7): at a split go left iff
 *   x[feature] < threshold; M(x) = base_score + sum over trees, in tree order, of the leaf
 *   reached, accumulated in fp32 one tree at a time.
 * Rejected with TP_EFORMAT: bad magic/version/size, a node index out of range, a cycle or a
 * shared or unreachable node, depth > max_depth, feature outside [-1, 3], a non-finite
 * threshold, a non-finite leaf or |leaf| > 2^60, a non-finite base, or more than 32767 distinct
 * thresholds on one feature.
 * tp_gbdt_load copies the normalised model to `device` (synchronously) and returns a handle.
 */
int tp_gbdt_load(const void* host_blob, size_t nbytes, int device, tp_gbdt** out);
int tp_gbdt_free(tp_gbdt* m);
int tp_gbdt_get_info(const tp_gbdt* m, tp_gbdt_info* out);

/*
 * K1 -- projection (Eq. 1-2) and FIFO admission (check 1 + batch cap, P:506-507,
 * P:755; reading A-2).
 *   inst    [dev] n_inst headers.            req  [dev] n_req entries (running then queued
 *                                                 per instance, at inst.req_begin).
 *   B, KV   [dev] out, int32 [n_inst][H]: B[i][m-1] = number of scheduled requests active at
 *           iteration m, KV[i][m-1] = sum of their Eq. 1 block counts
 *           ceil((a + m - 1 + q) / N) (0 beyond each request's l); zero for m > n.
 *           "Scheduled" = running + admitted queued.
 *   n       [dev] out, int32 [n_inst]: horizon = max l over scheduled requests (0 if none).
 *   n_adm   [dev] out, int32 [n_inst]: queued requests admitted (a FIFO prefix).
 *   status  [dev] out, uint32 [n_inst]: written (not OR-ed) with BAD_INPUT, EMPTY,
 *           BYPASS_LOST, KV_OVER, QUEUE_BLOCKED.
 * Admission: queued c (in order) is admitted iff B[1] + 1 <= max_batch and
 *   max_m (KV[m] + ceil((m - 1 + q_c) / N) [m <= r_c]) <= kv_cap; the first failure stops the
 *   queue and sets QUEUE_BLOCKED.
 */
int tp_project(const tp_inst* inst, int32_t n_inst, const tp_req* req, int32_t n_req, int32_t H,
               int32_t* B, int32_t* KV, int32_t* n, int32_t* n_adm, uint32_t* status, void* stream);

/*
 * K2 -- GBDT IPS model on the grid.  For every instance i not flagged
 * BAD_INPUT / EMPTY / BYPASS_LOST in status[i], every level u < F and every m = 1..n[i]:
 *   raw = M(tp_i, B[i][m-1], KV[i][m-1], freq_mhz[u])      (features as fp32)
 *   ips[(i*F + u)*H + m-1] = clamp(raw)  with NaN -> 2^-4, then [2^-4, 2^17] (reading A-8),
 * OR-ing TP_ST_IPS_CLAMPED into status[i] if any value was changed by the clamp.
 * Entries with m > n[i] and skipped instances are not written.
 *   freq_mhz [host] F levels, strictly ascending, finite, > 0 (reading A-19).
 *   ips      [dev] out, fp32 [n_inst][F][H].
 */
int tp_predict_ips(const tp_gbdt* m, const tp_inst* inst, int32_t n_inst, const int32_t* B,
                   const int32_t* KV, const int32_t* n, int32_t H, const float* freq_mhz, int32_t F,
                   float* ips, uint32_t* status, void* stream);

/*
 * K2, run-compressed (same outputs, bit for bit, as tp_predict_ips).  M depends on the iteration
 * m only through the features (B[m], KV[m]) and, for a given ensemble, only through their ranks
 * among the ensemble's thresholds; consecutive iterations with equal ranks ("runs", typically
 * 5-10 iterations long: KV grows by about B/N blocks per iteration) therefore share one IPS value
 * exactly.  A first kernel builds each instance's runs; the ensemble is then evaluated once per
 * (run, level) -- or, in cell mode, once per distinct (rank_tp, rank_B, rank_KV) cell and level
 * across the whole batch into a lookup table that a last kernel expands onto every iteration.
 *   workspace [dev] scratch owned by the caller, not used concurrently by another call:
 *             >= tp_predict_ips_workspace_size(m, n_inst, H, F) bytes enables cell mode (used when
 *             the model's dense cell space (n_cuts[0]+1)(n_cuts[1]+1)(n_cuts[2]+1) <= 2^22);
 *             >= tp_predict_ips_workspace_size(NULL, n_inst, H, F) bytes gives run mode.
 *   ips       [dev] as tp_predict_ips; may be NULL in cell mode (values stay in the workspace for
 *             tp_select_freq_ws; IPS_CLAMPED is then set by tp_select_freq_ws).
 * Other arguments, outputs and errors: as tp_predict_ips.
 */
size_t tp_predict_ips_workspace_size(const tp_gbdt* m, int32_t n_inst, int32_t H, int32_t F);
int tp_predict_ips_runs(const tp_gbdt* m, const tp_inst* inst, int32_t n_inst, const int32_t* B,
                        const int32_t* KV, const int32_t* n, int32_t H, const float* freq_mhz,
                        int32_t F, float* ips, uint32_t* status, void* workspace,
                        size_t workspace_bytes, void* stream);

/* Diagnostics (synchronous, not for the hot path): total number of runs the last
 * tp_predict_ips_runs call on `workspace` evaluated (per level). */
int tp_runs_total(const void* workspace, int32_t n_inst, int32_t H, int64_t* total);
/* ... and the number of distinct cells evaluated in cell mode (0 in run mode); `workspace` sized
 * by tp_predict_ips_workspace_size(m, n_inst, H, F). */
int tp_cells_total(const tp_gbdt* m, const void* workspace, int32_t n_inst, int32_t H, int32_t F,
                   int64_t* total);

/*
 * K3 -- SLO scan and frequency choice (Eq. 3-4; throttle P:550-557).
 * For each instance not flagged BAD_INPUT / EMPTY / BYPASS_LOST and each level u:
 *   T'[m] = fl32(1 / ips[m])                                       (reading A-9)
 *   T_R[l] = sum_{m <= l} T'[m], exactly, as int64 ticks of 2^-40 s  (Eq. 3, reading A-10)
 *   pass_u = T_R[n] <= n * tbt_slo                                  (TBT, tie passes)
 *            and T_R[l_j] < fl64(t_dead_j - t_cur) for every scheduled request j
 *                                                                   (Eq. 4 strict, A-12)
 *   level[i] = min{u : pass_u}, else F-1 with INFEASIBLE.  BAD_INPUT -> F-1, EMPTY -> 0,
 *   BYPASS_LOST -> F-1.
 *   req, t_dead [dev] the same request array as tp_project; t_dead fp64 seconds per entry.
 *   n, n_adm    [dev] from tp_project.   ips [dev] from tp_predict_ips.
 *   level       [dev] out, int32 [n_inst], an index into the frequency list.
 *   status      [dev] in/out: INFEASIBLE is OR-ed in.
 *   tr_ticks    [dev] optional out, int64 [n_inst][F][H] (m <= n, evaluated instances), or NULL.
 */
int tp_select_freq(const tp_inst* inst, int32_t n_inst, const tp_req* req, int32_t n_req,
                   const double* t_dead, const int32_t* n, const int32_t* n_adm, const float* ips,
                   int32_t H, int32_t F, float tbt_slo, int32_t* level, uint32_t* status,
                   int64_t* tr_ticks, void* stream);

/*
 * K3 fused with K2's cell mode: after tp_predict_ips_runs(m, ..., ips = NULL, workspace) in cell mode
 * the IPS values live only in the workspace's per-cell table; this K3 reads them through each
 * instance's runs (same outputs as tp_select_freq on the expanded grid, bit for bit), so the
 * [n_inst][F][H] ips grid is never written or read.  TP_ST_IPS_CLAMPED is OR-ed here.
 * TP_EINVAL if the workspace / model has no cell mode or H > 8192.  Other arguments: as
 * tp_select_freq.
 */
int tp_select_freq_ws(const tp_gbdt* m, const void* workspace, const tp_inst* inst, int32_t n_inst,
                      const tp_req* req, int32_t n_req, const double* t_dead, const int32_t* n,
                      const int32_t* n_adm, int32_t H, int32_t F, float tbt_slo, int32_t* level,
                      uint32_t* status, int64_t* tr_ticks, void* stream);

/*
 * K3 in the paper's search order (PAPER §4.5; reading A-24): the binary
 * search over the frequency range instead of the exhaustive scan.  Same inputs, outputs, LUT
 * workspace and errors as tp_select_freq_ws, without the T_R output.  Per instance: the top level
 * F-1 is checked (fails -> level F-1 + INFEASIBLE); then lo = 0, hi = F-1, and while lo < hi,
 * mid = (lo + hi) / 2 moves hi to mid if mid passes, lo to mid + 1 otherwise; level = lo.
 * IPS_CLAMPED covers the visited levels only.  Equals tp_select_freq_ws whenever the pass/fail
 * outcome is monotone in the level; otherwise the answer is the one the paper's search reaches.
 * The search is unrolled speculatively on the GPU (one warp per candidate level, 8 per round);
 * only the levels on the search path affect the result.
 */
int tp_select_freq_binary(const tp_gbdt* m, const void* workspace, const tp_inst* inst, int32_t n_inst,
                          const tp_req* req, int32_t n_req, const double* t_dead, const int32_t* n,
                          const int32_t* n_adm, int32_t H, int32_t F, float tbt_slo, int32_t* level,
                          uint32_t* status, void* stream);

/*
 * The compact path ("fused round"): the same decisions as K1 -> K2 -> K3 above, bit
 * for bit, with the per-iteration curves kept on chip.  Three kernels on one cell-mode workspace
 * (tp_predict_ips_workspace_size(m, n_inst, H, F) bytes; the model's cell space must be <= 2^22):
 *
 * tp_project_compact -- K1c, one warp per instance: tp_project's projection + FIFO gate (same
 *   n / n_adm / status outputs), then, for every instance not flagged BAD_INPUT / EMPTY /
 *   BYPASS_LOST, (a) the runs of consecutive iterations m <= n in one cell (rank_tp, rank_B[m],
 *   rank_KV[m]) of the ensemble's thresholds, first-seen cells claimed in the workspace's cell
 *   table, and (b) the deadline list of Eq. 4: for each end position l of a scheduled
 *   (running or admitted) request, Dmin[l] = min ceil(fl64(t_dead - t_cur) * 2^40) (reading A-12).
 *   B / KV [dev] optional (both NULL or both set): full [n_inst][H] rows as tp_project if
 *   bkv_rows = 1, only the m = 1 column (B[i*H], KV[i*H]) if bkv_rows = 0.
 *   t_dead [dev] fp64 seconds per request entry (as tp_select_freq).  H <= 16384 (the per-warp
 *   shared histograms fit up to H = 16384; larger H fails the general H check with TP_EINVAL).
 * tp_predict_cells -- K2 on the claimed cells: LUT[cell][u] = clamp(M(cell, freq_mhz[u])) (as
 *   tp_predict_ips_runs in cell mode; no pre-pass: the runs come from tp_project_compact).
 * tp_select_freq_compact -- K3c, one warp per instance, lane u = level u: T_R formed run by run
 *   from the LUT (exact ticks), Eq. 4 checked at the deadline list, TBT at m = n; level = lowest
 *   passing level (search = TP_SEARCH_EXHAUSTIVE, reading A-13) or the paper's binary search on the
 *   pass bits (TP_SEARCH_BINARY, reading A-24; IPS_CLAMPED then covers the visited levels only).
 *   Outputs and the BAD_INPUT / EMPTY / BYPASS_LOST / INFEASIBLE rules: as tp_select_freq.
 * All three: asynchronous on `stream`; TP_EINVAL on bad arguments or a too-small workspace.
 */
int tp_project_compact(const tp_gbdt* m, void* workspace, size_t workspace_bytes, const tp_inst* inst,
                       int32_t n_inst, const tp_req* req, int32_t n_req, const double* t_dead, int32_t H,
                       int32_t* B, int32_t* KV, int32_t bkv_rows, int32_t* n, int32_t* n_adm,
                       uint32_t* status, void* stream);
int tp_predict_cells(const tp_gbdt* m, void* workspace, size_t workspace_bytes, int32_t n_inst, int32_t H,
                     const float* freq_mhz, int32_t F, void* stream);
int tp_select_freq_compact(const tp_gbdt* m, const void* workspace, size_t workspace_bytes, int32_t n_inst,
                           const int32_t* n, int32_t H, int32_t F, float tbt_slo, int32_t search,
                           int32_t* level, uint32_t* status, void* stream);

/* Statistics of the last tp_project_compact on `workspace` (host copies; synchronises the device):
 * out[0] = pieces over all instances (the records K1c wrote and K3c walks), out[1] = end positions
 * (iterations where a scheduled request finishes), out[2] = distinct cells claimed (LUT rows K2
 * evaluates).  For measurement (bench.py's algorithmic byte counts), not on the decision path. */
int tp_compact_stats(const tp_gbdt* m, const void* workspace, size_t workspace_bytes, int32_t n_inst,
                     int32_t H, int32_t F, int64_t* out);

/*
 * Convenience: one decision round with library-owned scratch.
 * tp_ctx_create allocates, on `device`, B/KV/n/n_adm (n_inst_max x H), the ips grid
 * (n_inst_max x F_max x H), the K2 workspace (sized for `model`'s cell mode; NULL = run mode)
 * and staging for up to n_req_max requests.
 */
typedef struct tp_ctx tp_ctx;
int tp_ctx_create(int device, const tp_gbdt* model, int32_t n_inst_max, int32_t n_req_max, int32_t H,
                  int32_t F_max, tp_ctx** out);
int tp_ctx_free(tp_ctx* c);

/* K1 -> K2 -> K3 on device-resident inputs; level/status [dev] out.  tp_decide, tp_decide_host
 * and tp_decide_admit make the context's device current for the call and restore the caller's.  With TP_K2_COMPACT (the default
 * for a context created for `m`) the compact path runs: tp_project_compact (B/KV: m = 1 column only)
 * -> tp_predict_cells -> tp_select_freq_compact.  With TP_K2_RUNS (the default otherwise) and a
 * context created for `m`, K2 runs in cell mode without materialising the ips grid
 * (tp_predict_ips_runs with ips = NULL, then tp_select_freq_ws); without the model, run mode and
 * tp_select_freq.  TP_K2_COMPACT without the context's model -> TP_ENOTIMPL. */
int tp_decide(tp_ctx* c, const tp_gbdt* m, const tp_inst* inst, int32_t n_inst, const tp_req* req,
              int32_t n_req, const double* t_dead, const float* freq_mhz, int32_t F, float tbt_slo,
              int32_t* level, uint32_t* status, void* stream);

/* Same with HOST inputs/outputs: enqueues host->device copies of inst/req/t_dead, the three
 * kernels and device->host copies of level/status, all on `stream`.  Outputs are valid after
 * the stream is synchronised.  Use pinned host memory for asynchronous copies.  When the host
 * inputs are packed back to back (h_req == (char*)h_inst + n_inst * sizeof(tp_inst) and h_t_dead ==
 * (char*)h_req + n_req * sizeof(tp_req)) they travel in ONE copy, and when h_status == h_level +
 * n_inst the outputs come back in one copy. */
int tp_decide_host(tp_ctx* c, const tp_gbdt* m, const tp_inst* h_inst, int32_t n_inst,
                   const tp_req* h_req, int32_t n_req, const double* h_t_dead,
                   const float* freq_mhz, int32_t F, float tbt_slo, int32_t* h_level,
                   uint32_t* h_status, void* stream);

/*
 * Full admission control (PAPER §4.3.2) followed by the throttle.
 * Queued requests are considered in FIFO order, one at a time, at most q_max per decision
 * (reading A-23): a candidate is admitted iff, with it virtually appended, check 1 (KV
 * capacity + batch cap) holds, check 2 (mean TBT at the maximum frequency)
 * holds and check 3 (Eq. 4 at the maximum frequency) holds for every non-lost scheduled
 * request; if check 3 fails only for the candidate itself it is admitted as "lost" and
 * later checks ignore it; otherwise the queue stops.  Then levels are chosen as by tp_decide (a
 * lost request present -> maximum frequency).
 * tp_ctx_enable_admission(c, q_max) allocates the per-prefix scratch (q_max <= 32; the context must
 * have been created for `m`, H <= 8192).
 *   n_adm_out    [dev] optional int32 [n_inst]: queued requests admitted.
 *   adm_lost_out [dev] optional uint32 [n_inst]: bit c = the c-th queued request admitted as lost
 *                (the caller persists TP_REQ_LOST on it).
 */
int tp_ctx_enable_admission(tp_ctx* c, int32_t q_max);
int tp_decide_admit(tp_ctx* c, const tp_gbdt* m, const tp_inst* inst, int32_t n_inst, const tp_req* req,
                    int32_t n_req, const double* t_dead, const float* freq_mhz, int32_t F, float tbt_slo,
                    int32_t* level, uint32_t* status, int32_t* n_adm_out, uint32_t* adm_lost_out,
                    void* stream);

/* Which path tp_decide / tp_decide_host use (default TP_K2_COMPACT for a context created for a model
 * with a cell mode, TP_K2_RUNS otherwise). */
enum { TP_K2_DIRECT = 0, TP_K2_RUNS = 1, TP_K2_COMPACT = 2 };
int tp_ctx_set_k2_mode(tp_ctx* c, int mode);   /* may allocate the ips grid: TP_ENOMEM */

/* K3 search order for tp_decide / tp_decide_host / tp_decide_admit (default exhaustive, reading
 * A-13).  TP_SEARCH_BINARY (reading A-24) is supported by the compact path (TP_K2_COMPACT, the
 * default: K3c replays the search on its per-level pass bits) and by the fused cell path
 * (TP_K2_RUNS with a context created for the model and H <= 8192, tp_select_freq_binary); with
 * TP_K2_DIRECT, or TP_K2_RUNS without a cell-mode model, those calls return TP_ENOTIMPL. */
enum { TP_SEARCH_EXHAUSTIVE = 0, TP_SEARCH_BINARY = 1 };
int tp_ctx_set_search(tp_ctx* c, int search);

/* Device pointers of the context's scratch (for inspection / tests); any out may be NULL.  After a
 * TP_K2_COMPACT tp_decide only the m = 1 column of B / KV is written, and ips is not (a context
 * created for a cell-mode model allocates the ips grid only when tp_ctx_set_k2_mode selects a
 * mode that writes it; before that, *ips is NULL). */
int tp_ctx_buffers(tp_ctx* c, int32_t** B, int32_t** KV, int32_t** n, int32_t** n_adm, float** ips);

/*
 * Trace replay (BASELINE configs[3]): advance every instance by one engine
 * iteration after a decision round, on the GPU.  The request table uses fixed slots: instance i owns
 * req[i * slot_cap .. (i + 1) * slot_cap) (inst[i].req_begin must be i * slot_cap), running entries
 * first, then the FIFO queue.  For each instance with n > 0 the iteration lasts
 * T' = fl32(1 / clamp(M(tp, B[1], KV[1], freq_mhz[level]))) seconds (the Scheduler's own time
 * model): t_cur += T', k += 1; every scheduled request (running + the n_adm admitted
 * queued ones) emits one token (a += 1) and completes when a == r (struck; oracle
 * length predictor); the rest of the queue stays.  An idle instance (n = 0) jumps its
 * clock to its next arrival.  Arrivals (per instance, sorted by time: arr_t[arr_off[i] ..
 * arr_off[i+1]), records arr_req with deadlines arr_dead) with arr_t <= the new clock join the
 * queue tail, up to slot_cap (the rest are dropped).  BAD_INPUT instances are left as they are.
 *   inst [dev] in/out (n_run, n_queue, k, t_cur);  req, t_dead [dev] in;  req_out, t_dead_out
 *   [dev] out (same slot layout; the caller swaps the buffers);  B, KV, n, n_adm, status, level
 *   [dev] the round's K1 / K3 outputs;  freq_mhz [host] the round's levels;  arr_next [dev] in/out
 *   next arrival per instance;  stats [dev] uint64[5] accumulators: completed, completed before
 *   their deadline (Eq. 4), dropped arrivals, engine iterations, admissions;  adm_lost [dev]
 *   optional (tp_decide_admit's output): admitted queued requests marked lost get TP_REQ_LOST.
 */
int tp_replay_advance(const tp_gbdt* m, tp_inst* inst, int32_t n_inst, const tp_req* req,
                      const double* t_dead, tp_req* req_out, double* t_dead_out, int32_t slot_cap,
                      int32_t H, const int32_t* B, const int32_t* KV, const int32_t* n,
                      const int32_t* n_adm, const uint32_t* status, const int32_t* level,
                      const float* freq_mhz, int32_t F, const double* arr_t, const tp_req* arr_req,
                      const double* arr_dead, const int64_t* arr_off, int64_t* arr_next,
                      uint64_t* stats, const uint32_t* adm_lost, void* stream);

const char* tp_strerror(int code);
int tp_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TP_H */
