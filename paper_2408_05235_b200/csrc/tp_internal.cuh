// Internal declarations shared by libtp's translation units (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "tp.h"

namespace tp {

constexpr int kMaxF = 32;
constexpr int kMaxH = 16384;
constexpr int kMaxHRunsSelect = 8192;      // tp_select_freq_ws keeps ~28 B per iteration in smem
constexpr int kMaxDepth = 12;
constexpr uint64_t kMaxModelWords = 1ull << 28;   // node words of a loaded ensemble (1 GiB)
constexpr int kMaxCuts = 32767;            // ranks must fit 15 bits (K2 word encoding)
constexpr int64_t kFeatLimit = 1LL << 24;  // integer features exact in fp32
constexpr int kRankTabMax = 1 << 16;       // rank table entries per integer feature

// Unsigned division by a run-time invariant d >= 1, exact for every 32-bit dividend (Granlund &
// Montgomery, "Division by invariant integers using multiplication", 1994, Fig. 4.1):
// l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1, q = (t + ((n - t) >> min(l,1))) >> max(l-1,0),
// t = mulhi(m, n).  Used by K1 for the per-instance block size N.
struct FastDiv {
    uint32_t m, s1, s2;
    FastDiv() = default;
    __host__ __device__ explicit FastDiv(uint32_t d) {
#ifdef __CUDA_ARCH__
        const uint32_t l = d > 1 ? 32 - __clz(d - 1) : 0;   // ceil(log2 d)
#else
        uint32_t l = 0;
        while (l < 32 && (1ull << l) < d) ++l;
#endif
        m = (uint32_t)((((1ull << l) - d) << 32) / d + 1);
        s1 = l < 1 ? l : 1;
        s2 = l > 1 ? l - 1 : 0;
    }
#ifdef __CUDACC__
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        const uint32_t t = __umulhi(m, n);
        return (t + ((n - t) >> s1)) >> s2;
    }
#endif
};

// Device-resident, normalised ensemble (built by tp_gbdt_load, model.cu).
//
// Node words: tree t occupies words[t * TW .. (t + 1) * TW), TW = max(4, 2 << D), a complete binary heap
// with 1-based index: internal node idx in [1, 2^D), leaf idx in [2^D, 2^(D+1)), children of idx at
// 2*idx (left, x < thr) and 2*idx + 1.  word 0 is unused.
//   internal word = ((0xFFFF - j) << 16) | sel(f)
//     f   = split feature, j = index of the threshold among feature f's sorted distinct cuts;
//     sel = PRMT selector moving rank_f (16 bits at byte 2f of the 8-byte feature pair) into the
//           upper half: bytes (b1, b1, b0, b1) with b0 = 2f, b1 = 2f + 1.
//     K2 computes r = prmt(xlo, xhi, word) = rank_f << 16 | junk (junk <= 0x7F7F) and
//     go_right = carry_out(r + word)  <=>  rank_f + 0xFFFF - j >= 0x10000  <=>  rank_f > j
//                                      <=>  x_f >= cut_j  (rank = #cuts <= x).
//   leaf word = bit pattern of the fp32 leaf value.
// Shallow leaves are replicated down to depth D (exactly equivalent).
struct Model {
    int device = 0;
    int32_t n_trees = 0, depth = 0;
    float base = 0.f;
    int32_t n_cuts[4] = {0, 0, 0, 0};
    uint32_t* d_words = nullptr;   // n_trees * (2 << depth)
    float* d_cuts = nullptr;       // concatenated sorted cuts, feature order
    int32_t cut_off[5] = {0, 0, 0, 0, 0};
    // rank tables for the integer features batch (0) and KV (1): rank(x) = rtab[off + x] for
    // 0 <= x < len (len <= 65536; beyond it, a binary search over the cuts)
    uint16_t* d_rtab = nullptr;
    int32_t rtab_off[2] = {0, 0}, rtab_len[2] = {0, 0};
    int64_t device_bytes = 0;
    // 8 when every possible output of the ensemble lies in (1, 512) IPS (bounded at load from the
    // leaves): then every T' = fl32(1/ips) lies in (2^-9, 1) s, so its tick count is a multiple of
    // 2^8 below 2^40 and K2 can store T' / 2^8 ticks in 32 bits, exactly (compact path); else 0
    int32_t tick_shift = 0;
};

struct K2Params {
    const uint32_t* words;
    const float* cuts;
    int32_t cut_off[5];
    int32_t n_trees, depth;
    float base;
    const tp_inst* inst;
    const int32_t* B;
    const int32_t* KV;
    const int32_t* n;
    uint32_t* status;
    float* ips;
    int32_t n_inst, H, F;
    uint32_t skip;           // status bits of instances K2 does not evaluate
    float freq[kMaxF];
    const uint16_t* rtab;
    int32_t rtab_off[2], rtab_len[2];
    // run-compressed mode (tp_predict_ips_runs): consecutive iterations with identical
    // (batch, KV) threshold ranks form a run; the ensemble is evaluated once per run.
    int32_t* run_h;          // [n_inst] runs per instance (0 for skipped instances)
    int32_t* run_m;          // [n_inst][H] first iteration m of each run
    uint32_t* run_key;       // [n_inst][H] rank_B | rank_KV << 16 of each run (cell id in cell mode)
    // cell-memoised mode: M depends on a grid row only through its cell = (rank_tp, rank_B,
    // rank_KV) (and the level); distinct cells are evaluated once into a LUT, then expanded.
    int32_t* cell_tab;       // [n_cells] dense cell id -> LUT row (-1 = absent), or null
    uint32_t* cell_list;     // [cap] LUT row -> cell id
    int32_t* cell_count;     // [1] distinct cells - 1 (directly before cell_tab: one reset for both)
    float* lut;              // [cap][F] clamped IPS
    long long* lut_ticks;    // [n_cells][F] by cell id: T' = fl32(1 / ips) in ticks of 2^-40 s (A-9, A-10)
    uint32_t* cell_clamp;    // [n_cells] by cell id: bit u set if level u's value was clamped
    int32_t n_cells, cell_cap;
    // compact path (K1c -> K2 cells -> K3c): K1c already built the runs and claimed the cells, so
    // the K2 launch skips its k2_runs pre-pass and the cell-table resets
    int32_t runs_ready;
    // compact path: the model's tick_shift; with 8, lut_ticks holds uint32 T' / 2^8 tick values
    // and K1c's Dmin / K3c's T_R count units of 2^8 ticks (2^-32 s)
    int32_t tick_shift;
    // compact path: run_h / run_m / run_key hold K1c's PIECES (k1_compact.cu, piece_rules), end_d
    // each piece's Dmin in ticks of 2^-40 s (reading A-12; INT64_MAX: no deadline), end_n the
    // number of end positions (statistics); written by K1c, read by K3c
    int32_t* end_n;          // [n_inst]
    long long* end_d;        // [n_inst][H]
    // compact path, K1c's packed histograms: instances that do not fit them (count - 1, directly
    // before cell_count: reset by the same memset) and their list, handled by the wide kernel
    int32_t* flag_count;
    int32_t* flag_list;      // [n_inst]
    // compact path, K3c's persistent warps: next instance and finished CTAs (count - 1; reset by
    // K1c's memset and re-armed by K3c's last CTA)
    int32_t* k3_next;
    int32_t* k3_done;
    int32_t* k1_next;        // K1c (packed, persistent warps): next instance (count - 1)
};

// workspace for tp_predict_ips_runs; cell mode is used when the model's dense cell space
// (nTP+1)(nB+1)(nKV+1) is at most kMaxCells
constexpr int64_t kMaxCells = 1LL << 22;
size_t runs_workspace_bytes(int64_t n_cells, int32_t n_inst, int32_t H, int32_t F);
void runs_workspace_carve(void* ws, int64_t n_cells, int32_t n_inst, int32_t H, int32_t F, K2Params& p);
int64_t model_cells(const Model& m);

#ifdef __CUDACC__
// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl may start while the
// previous kernel on the stream drains; it must execute pdl_wait() before touching anything the
// previous kernel writes (a no-op when launched without the attribute).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// One warp's own hardware barrier (named barrier `id` in [1, 15], 32 threads).  Used where a
// warp hands data to itself through shared memory inside a persistent loop (ids 1..15): a __syncwarp() that
// the compiler considers redundant is emitted as nothing, and the lanes are then not reliably
// reconverged (measured on B200: stale shared-memory reads).  The ids are immediates so that ptxas
// reserves only the barriers actually used (a register id reserves all 16 and caps occupancy).
__device__ __forceinline__ void warp_bar(int id) {
    switch (id) {
        case 1: asm volatile("bar.sync 1, 32;" ::: "memory"); break;
        case 2: asm volatile("bar.sync 2, 32;" ::: "memory"); break;
        case 3: asm volatile("bar.sync 3, 32;" ::: "memory"); break;
        case 4: asm volatile("bar.sync 4, 32;" ::: "memory"); break;
        case 5: asm volatile("bar.sync 5, 32;" ::: "memory"); break;
        case 6: asm volatile("bar.sync 6, 32;" ::: "memory"); break;
        case 7: asm volatile("bar.sync 7, 32;" ::: "memory"); break;
        case 8: asm volatile("bar.sync 8, 32;" ::: "memory"); break;
        case 9: asm volatile("bar.sync 9, 32;" ::: "memory"); break;
        case 10: asm volatile("bar.sync 10, 32;" ::: "memory"); break;
        case 11: asm volatile("bar.sync 11, 32;" ::: "memory"); break;
        case 12: asm volatile("bar.sync 12, 32;" ::: "memory"); break;
        case 13: asm volatile("bar.sync 13, 32;" ::: "memory"); break;
        case 14: asm volatile("bar.sync 14, 32;" ::: "memory"); break;
        default: asm volatile("bar.sync 15, 32;" ::: "memory"); break;
    }
}

// &base[idx] for a 32-bit unsigned index as ONE IMAD.WIDE.U32 (nvcc otherwise often widens the
// index and adds it with carries, 3-5 instructions per address)
template <typename T>
__device__ __forceinline__ T* ptr_at(T* base, unsigned idx) {
    T* a;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a) : "r"(idx), "n"((int)sizeof(T)), "l"(base));
    return a;
}

// Bulk L2 prefetch of [p, p + bytes) (p 16-byte aligned, bytes a multiple of 16): one instruction
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

constexpr long long kNoDeadline = 0x7fffffffffffffffLL;
// ceil(s * 2^40) for the E2E compare T_R < s (T_R integer ticks of 2^-40 s, reading A-12):
// <= 0 / NaN -> 0 (never passes), >= 2^62 -> INT64_MAX (always passes; T_R < 2^58).
__device__ __forceinline__ long long slack_ticks(double s, int shift = 0) {
    const double d = s * (shift ? 0x1p32 : 0x1p40);   // units of 2^shift ticks (shift 0 or 8)
    if (!(d > 0.0)) return 0;
    if (d >= 0x1p62) return kNoDeadline;
    return (long long)ceil(d);
}
// T' of one IPS value in ticks of 2^-40 s: fl32 reciprocal (reading A-9), exact scaling.
__device__ __forceinline__ long long ticks_of(float ips) {
    const float t = __frcp_rn(ips);
    return (long long)(t * 0x1p40f);    // exact: t in [2^-17, 16]
}
#endif

// Compact path.  K1c: projection + FIFO gate (as launch_project) + run compression, cell claims
// and the per-instance deadline list, one warp per instance.  `w` carries the model's cut / rank
// tables and the workspace (cell mode required).  B/KV: NULL, m = 1 only (bkv_rows = 0) or full
// rows (bkv_rows = 1).
int launch_project_compact(const K2Params& w, const tp_inst* inst, int32_t n_inst, const tp_req* req,
                           int32_t n_req, const double* t_dead, int32_t H, int32_t* B, int32_t* KV, int bkv_rows,
                           int32_t* n, int32_t* n_adm, uint32_t* status, uint32_t skip, cudaStream_t s,
                           const int32_t* force_adm = nullptr, const uint32_t* lost_mask = nullptr);
// K3c: one warp per instance, lane u = level u; T_R formed run by run from the LUT, checked at the
// deadline list's end positions; search 0 = exhaustive (A-13), 1 = the paper's binary search (A-24).
int launch_select_compact(const K2Params& w, int32_t n_inst, const int32_t* n, int32_t H, int32_t F,
                          int64_t tbt_ticks, int search, uint32_t skip, int32_t* level, uint32_t* status,
                          cudaStream_t s);
// K1c's shared memory per warp for horizon H (bytes)
int project_compact_smem_per_warp(int32_t H);

int launch_project(const tp_inst* inst, int32_t n_inst, const tp_req* req, int32_t n_req, int32_t H,
                   int32_t* B, int32_t* KV, int32_t* n, int32_t* n_adm, uint32_t* status, cudaStream_t s,
                   const int32_t* force_adm = nullptr, const uint32_t* lost_mask = nullptr);
int launch_gbdt(const K2Params& p, bool runs, cudaStream_t s);
int launch_select(const tp_inst* inst, int32_t n_inst, const tp_req* req, int32_t n_req, const double* t_dead,
                  const int32_t* n, const int32_t* n_adm, const float* ips, int32_t H, int32_t F,
                  int64_t tbt_ticks, int32_t* level, uint32_t* status, int64_t* tr, const K2Params* ws,
                  int search, cudaStream_t s);

int launch_replay_advance(const Model& m, tp_inst* inst, int32_t n_inst, const tp_req* req, const double* t_dead,
                          tp_req* req_out, double* t_dead_out, int32_t cap, int32_t H, const int32_t* B,
                          const int32_t* KV, const int32_t* n, const int32_t* n_adm, const uint32_t* status,
                          const int32_t* level, const float* freq, int32_t F, const double* arr_t,
                          const tp_req* arr_req, const double* arr_dead, const int64_t* arr_off, int64_t* arr_next,
                          unsigned long long* stats, const uint32_t* adm_lost, cudaStream_t s);

int launch_admit_expand(const tp_inst* inst, int32_t n_inst, int32_t qc, const int32_t* n_adm1,
                        const uint32_t* status1, tp_inst* vinst, int32_t* vforce, cudaStream_t s);
int launch_admit_checks(const tp_inst* vinst, int32_t n_v, const tp_req* req, const double* t_dead,
                        const int32_t* vn, const uint32_t* vstatus, const K2Params& ws, int32_t H,
                        int64_t tbt_ticks, uint2* vres, cudaStream_t s);
int launch_admit_resolve(int32_t n_inst, int32_t qc, const tp_inst* inst, const uint32_t* status1,
                         const int32_t* n_adm1, const uint2* vres, int32_t* n_adm, uint32_t* lost, cudaStream_t s);

}  // namespace tp

struct tp_gbdt {
    tp::Model m;
};
