// Trace replay state advance (BASELINE configs[3]): after a decision round,
// advance every serving instance by one engine iteration at its chosen frequency, on the GPU.
//
// The engine model is the paper's own: an iteration takes T' = 1/IPS seconds with IPS predicted
// by M at the iteration's batch size, KV usage and the chosen frequency (the Scheduler's
// time model; "oracle" length predictor: a request completes exactly after r^ tokens);
// every scheduled request emits one token per iteration; a completed request is struck
// from the Scoreboard; admitted queued requests start this iteration (virtual append at
// s = k committed); arrivals join the FIFO queue when the clock passes their arrival time.
//
// One CTA per instance.  The request table uses fixed slots: instance i owns
// req[i * cap .. (i + 1) * cap) (running first, then queued), so no global repacking is needed;
// the new table is written to a second buffer (double-buffered by the caller).
#include "tp_internal.cuh"

namespace tp {
namespace {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kSkip = TP_ST_BAD_INPUT;

__device__ __forceinline__ uint32_t rank_g(const float* __restrict__ c, int cnt, float x) {
    int lo = 0, hi = cnt;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(c + mid) <= x) lo = mid + 1;
        else hi = mid;
    }
    return (uint32_t)lo;
}

__device__ __forceinline__ uint32_t prmt_(uint32_t lo, uint32_t hi, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(lo), "r"(hi), "r"(sel));
    return r;
}

// block-wide exclusive scan of one int per thread (kThreads threads); returns (excl, total)
__device__ __forceinline__ int2 block_scan(int v, int* sw) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sw[warp] = x;
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        before += (w < warp) ? sw[w] : 0;
        total += sw[w];
    }
    __syncthreads();
    return make_int2(before + x - v, total);
}

struct AdvParams {
    const uint32_t* words;
    const float* cuts;
    int32_t cut_off[5];
    int32_t n_trees, depth, TW;
    float base;
    tp_inst* inst;
    const tp_req* req;
    const double* t_dead;
    tp_req* req_out;
    double* t_dead_out;
    int32_t n_inst, cap, H, F;
    const int32_t *B, *KV, *n, *n_adm, *level;
    const uint32_t* status;
    float freq[kMaxF];
    const double* arr_t;
    const tp_req* arr_req;     // {a = 0, q, r, flags}
    const double* arr_dead;
    const int64_t* arr_off;
    int64_t* arr_next;
    unsigned long long* stats;  // [completed, met, dropped, iterations, admitted]
    const uint32_t* adm_lost;   // optional: admitted queued requests marked lost (tp_decide_admit)
};

__global__ void __launch_bounds__(kThreads)
k_replay_advance(const __grid_constant__ AdvParams p) {
    __shared__ float s_leaf[1024];
    __shared__ int sw[kWarps];
    __shared__ double s_tnew;
    __shared__ int s_iter;
    const int i = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    tp_inst in = p.inst[i];
    const int64_t base = (int64_t)i * p.cap;
    const uint32_t st = p.status[i];
    const int nr = in.n_run, nq = in.n_queue;
    // tp_decide read this instance's requests at req_begin; the advance addresses slot i * cap:
    // the two must agree (include/tp.h), else the state is left as is (treated as bad input)
    const bool bad = (st & kSkip) != 0 || in.req_begin != base;
    const int n = bad ? 0 : p.n[i];
    const int nadm = bad ? 0 : p.n_adm[i];
    if (bad) {      // invalid instance data: state left as is
        for (int e = tid; e < nr + nq && e < p.cap; e += kThreads) {
            p.req_out[base + e] = p.req[base + e];
            p.t_dead_out[base + e] = p.t_dead[base + e];
        }
        return;
    }

    // ---- duration of this iteration: T' = fl32(1 / clamp(M(tp, B[1], KV[1], f_level))) ----
    if (tid < 32) {
        double t_new = in.t_cur;
        int iter = 0;
        if (n > 0) {
            const int u = p.level[i];
            const int b1 = p.B[(int64_t)i * p.H], kv1 = p.KV[(int64_t)i * p.H];
            const uint32_t xlo = rank_g(p.cuts + p.cut_off[0], p.cut_off[1] - p.cut_off[0], (float)in.tp) |
                                 (rank_g(p.cuts + p.cut_off[1], p.cut_off[2] - p.cut_off[1], (float)b1) << 16);
            const uint32_t xhi = rank_g(p.cuts + p.cut_off[2], p.cut_off[3] - p.cut_off[2], (float)kv1) |
                                 (rank_g(p.cuts + p.cut_off[3], p.cut_off[4] - p.cut_off[3], p.freq[u]) << 16);
            // lanes walk trees lane, lane + 32, ...; leaves are summed in tree order afterwards
            float acc = p.base;
            for (int t0 = 0; t0 < p.n_trees; t0 += 1024) {
                const int tn = min(1024, p.n_trees - t0);
                for (int t = lane; t < tn; t += 32) {
                    const uint32_t* tw = p.words + (size_t)(t0 + t) * p.TW;
                    uint32_t idx = 1;
                    for (int d = 0; d < p.depth; ++d) {
                        const uint32_t w = __ldg(tw + idx);
                        idx = 2 * idx + ((prmt_(xlo, xhi, w) > ~w) ? 1u : 0u);
                    }
                    s_leaf[t] = __uint_as_float(__ldg(tw + idx));
                }
                __syncwarp();
                if (lane == 0)
                    for (int t = 0; t < tn; ++t) acc = __fadd_rn(acc, s_leaf[t]);
                __syncwarp();
            }
            if (lane == 0) {
                const float ips = isnan(acc) ? 0x1p-4f : fminf(fmaxf(acc, 0x1p-4f), 0x1p17f);
                t_new = in.t_cur + (double)__frcp_rn(ips);
                iter = 1;
            }
        } else {
            // idle engine: the clock jumps to the next arrival (if any)
            const int64_t j = p.arr_next[i];
            if (lane == 0 && j < p.arr_off[i + 1] && p.arr_t[j] > t_new) t_new = p.arr_t[j];
        }
        if (lane == 0) {
            s_tnew = t_new;
            s_iter = iter;
        }
    }
    __syncthreads();
    const double t_new = s_tnew;
    const int iter = s_iter;

    // ---- survivors: running (+1 token), admitted queued (start now), remaining queue ----
    int nrun_new = 0, nq_keep = 0;
    unsigned long long completed = 0, met = 0;
    {
        const int n_sched = iter ? nr + nadm : 0;
        // pass 1: scheduled entries that survive the iteration keep their order as running
        for (int e0 = 0; e0 < n_sched; e0 += kThreads) {
            const int e = e0 + tid;
            bool keep = false;
            tp_req r{};
            double dl = 0;
            if (e < n_sched) {
                r = p.req[base + e];
                dl = p.t_dead[base + e];
                if (p.adm_lost && e >= nr && e - nr < 32 && ((p.adm_lost[i] >> (e - nr)) & 1u))
                    r.flags |= TP_REQ_LOST;                 // scheduled as "lost": persisted
                r.a += 1;                                   // one token generated this iteration
                if (r.r - r.a == 0) {                       // completes at the end of this iteration
                    ++completed;
                    met += t_new < dl;                       // Eq. 4 met (strict)
                } else {
                    keep = true;
                }
            }
            const int2 sc = block_scan(keep ? 1 : 0, sw);
            if (keep) {
                p.req_out[base + nrun_new + sc.x] = r;
                p.t_dead_out[base + nrun_new + sc.x] = dl;
            }
            nrun_new += sc.y;
        }
        // pass 2: queued requests not admitted stay queued, in FIFO order
        const int q0 = iter ? nr + nadm : nr;              // idle: nothing was admitted
        const int nrem = nr + nq - q0;
        for (int e0 = 0; e0 < nrem; e0 += kThreads) {
            const int e = e0 + tid;
            if (e < nrem) {
                p.req_out[base + nrun_new + e] = p.req[base + q0 + e];
                p.t_dead_out[base + nrun_new + e] = p.t_dead[base + q0 + e];
            }
        }
        nq_keep = nrem;
    }
    // ---- arrivals up to the new clock join the queue tail (dropped beyond the slot capacity) ----
    const int64_t a0 = p.arr_next[i], a1 = p.arr_off[i + 1];
    __syncthreads();
    int arrived = 0;
    {
        // count arrivals with t <= t_new (sorted); one warp scans ahead
        if (tid < 32) {
            int64_t j = a0;
            int cnt = 0;
            while (true) {
                const int64_t jj = j + lane;
                const bool in_ = jj < a1 && p.arr_t[jj] <= t_new;
                const unsigned b = __ballot_sync(0xffffffffu, in_);
                const int c = __popc(b);
                cnt += c;
                if (c < 32) break;
                j += 32;
            }
            if (lane == 0) sw[0] = cnt;
        }
        __syncthreads();
        arrived = sw[0];
        __syncthreads();
    }
    const int room = p.cap - (nrun_new + nq_keep);
    const int take = min(arrived, max(room, 0));
    for (int e = tid; e < take; e += kThreads) {
        tp_req r = p.arr_req[a0 + e];
        r.a = 0;
        p.req_out[base + nrun_new + nq_keep + e] = r;
        p.t_dead_out[base + nrun_new + nq_keep + e] = p.arr_dead[a0 + e];
    }
    // ---- header + statistics ----
    for (int o = 16; o; o >>= 1) {
        completed += __shfl_xor_sync(0xffffffffu, completed, o);
        met += __shfl_xor_sync(0xffffffffu, met, o);
    }
    if (lane == 0 && (completed | met)) {
        atomicAdd(p.stats + 0, completed);
        atomicAdd(p.stats + 1, met);
    }
    if (tid == 0) {
        in.n_run = nrun_new;
        in.n_queue = nq_keep + take;
        in.k += iter;
        in.t_cur = t_new;
        p.inst[i] = in;
        p.arr_next[i] = a0 + arrived;
        if (arrived > take) atomicAdd(p.stats + 2, (unsigned long long)(arrived - take));
        if (iter) atomicAdd(p.stats + 3, 1ull);
        if (iter && nadm) atomicAdd(p.stats + 4, (unsigned long long)nadm);
    }
}

}  // namespace

int launch_replay_advance(const Model& m, tp_inst* inst, int32_t n_inst, const tp_req* req, const double* t_dead,
                          tp_req* req_out, double* t_dead_out, int32_t cap, int32_t H, const int32_t* B,
                          const int32_t* KV, const int32_t* n, const int32_t* n_adm, const uint32_t* status,
                          const int32_t* level, const float* freq, int32_t F, const double* arr_t,
                          const tp_req* arr_req, const double* arr_dead, const int64_t* arr_off, int64_t* arr_next,
                          unsigned long long* stats, const uint32_t* adm_lost, cudaStream_t s) {
    if (n_inst == 0) return TP_OK;
    AdvParams p{};
    p.adm_lost = adm_lost;
    p.words = m.d_words;
    p.cuts = m.d_cuts;
    for (int f = 0; f < 5; ++f) p.cut_off[f] = m.cut_off[f];
    p.n_trees = m.n_trees;
    p.depth = m.depth;
    p.TW = (2 << m.depth) < 4 ? 4 : (2 << m.depth);
    p.base = m.base;
    p.inst = inst;
    p.req = req;
    p.t_dead = t_dead;
    p.req_out = req_out;
    p.t_dead_out = t_dead_out;
    p.n_inst = n_inst;
    p.cap = cap;
    p.H = H;
    p.F = F;
    p.B = B;
    p.KV = KV;
    p.n = n;
    p.n_adm = n_adm;
    p.level = level;
    p.status = status;
    for (int u = 0; u < F; ++u) p.freq[u] = freq[u];
    p.arr_t = arr_t;
    p.arr_req = arr_req;
    p.arr_dead = arr_dead;
    p.arr_off = arr_off;
    p.arr_next = arr_next;
    p.stats = stats;
    k_replay_advance<<<n_inst, kThreads, 0, s>>>(p);
    return cudaPeekAtLastError() == cudaSuccess ? TP_OK : TP_ECUDA;
}

}  // namespace tp
