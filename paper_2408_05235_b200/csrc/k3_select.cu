// K3 -- SLO scan and frequency choice: T' = 1/IPS, T_R = cumulative sum (Eq. 3),
// TBT check, E2E check Eq. 4, lowest SLO-meeting frequency with
// the lost bypass.
//
// One CTA per instance, one warp per frequency level (levels strided over the 8 warps).
//  * The scheduled requests' deadlines become a table Dmin[l] = min over requests ending at l of
//    ceil(fl64(t_dead - t_cur) * 2^40) (int64 ticks of 2^-40 s) in shared memory, so Eq. 4 for
//    every request is "T_R[l] < Dmin[l] at every end position l".
//  * T'[m] = fl32(1/ips) lies in [2^-17, 16] s, i.e. an integer number of 2^-40 s ticks, so T_R is
//    an exact int64 sum (reading A-10): any summation order gives the same bits, and the SLO
//    comparisons are exact integer compares.
//  * Only the lowest passing level matters: a warp skips a level above one that already passed,
//    and stops scanning a level at its first violated deadline (unless T_R is requested).
//
// k3_select      reads the [I][F][H] ips grid, one iteration per lane (tp_select_freq).
// k3_select_runs reads K2's cell LUT through the instance's runs (tp_select_freq_ws): on a run of
//                len iterations with constant T' = t, T_R grows by len * t (exact), so T_R is
//                formed per run and evaluated only at the requests' end positions.
#include "tp_internal.cuh"

namespace tp {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kSkip = TP_ST_BAD_INPUT | TP_ST_EMPTY | TP_ST_BYPASS_LOST;
// Per instance: dense Dmin table over m in [1, n] (shared memory).
__device__ __forceinline__ void build_dmin(long long* dmin, const tp_inst& in, int n_sched, int n,
                                           const int4* __restrict__ req, const double* __restrict__ t_dead) {
    for (int m = threadIdx.x; m <= n; m += kThreads) dmin[m] = kNoDeadline;
    __syncthreads();
    for (int e = threadIdx.x; e < n_sched; e += kThreads) {
        const int64_t j = (int64_t)in.req_begin + e;
        const int4 r = __ldg(&req[j]);
        const double slack = __ldg(&t_dead[j]) - in.t_cur;   // fl64(t_dead - t_cur), reading A-12
        atomicMin(&dmin[r.z - r.x], slack_ticks(slack));
    }
    __syncthreads();
}

__device__ __forceinline__ void finish(int i, int F, uint32_t st, uint32_t st_or, const int* s_pass,
                                       int32_t* level, uint32_t* status) {
    const int lane = threadIdx.x & 31;
    if ((threadIdx.x >> 5) != 0) return;
    const unsigned pass = __ballot_sync(0xffffffffu, lane < F && s_pass[lane]);
    if (lane == 0) {
        if (pass) {
            level[i] = __ffs(pass) - 1;
            if (st_or) status[i] = st | st_or;
        } else {
            level[i] = F - 1;
            status[i] = st | st_or | TP_ST_INFEASIBLE;
        }
    }
}

__global__ void __launch_bounds__(kThreads)
k3_select(const tp_inst* __restrict__ inst, const int4* __restrict__ req, const double* __restrict__ t_dead,
          const int32_t* __restrict__ nv, const int32_t* __restrict__ nadm, const float* __restrict__ ips,
          int32_t H, int32_t F, long long tbt_ticks, int32_t* __restrict__ level, uint32_t* __restrict__ status,
          long long* __restrict__ tr) {
    extern __shared__ long long dmin[];   // index m in [1, n]
    __shared__ int s_pass[kMaxF];
    __shared__ int s_best;
    const int i = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t st = status[i];
    if (st & kSkip) {
        if (tid == 0) level[i] = (st & TP_ST_BAD_INPUT) ? F - 1 : (st & TP_ST_EMPTY) ? 0 : F - 1;
        return;
    }
    const int n = nv[i];
    const tp_inst in = inst[i];
    if (tid < kMaxF) s_pass[tid] = 0;
    if (tid == 0) s_best = F;
    build_dmin(dmin, in, in.n_run + nadm[i], n, req, t_dead);

    const long long tbt_bound = (long long)n * tbt_ticks;   // TBT: T_R[n] <= n * slo (<= 2^58)
    for (int u = warp; u < F; u += kWarps) {
        if (!tr && u > *(volatile int*)&s_best) break;      // a lower level already passed
        const float* row = ips + ((size_t)i * F + u) * H;
        long long* trow = tr ? tr + ((size_t)i * F + u) * H : nullptr;
        long long carry = 0;
        bool ok = true;
        // 4 x 32 iterations per step: the 4 coalesced loads are issued back to back, then scanned
        for (int m0 = 1; m0 <= n; m0 += 128) {
            float v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int m = m0 + 32 * j + lane;
                v[j] = m <= n ? __ldg(row + m - 1) : 1.0f;
            }
            bool bad = false;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int m = m0 + 32 * j + lane;
                long long x = m <= n ? ticks_of(v[j]) : 0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const long long y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                const long long TR = carry + x;
                carry = __shfl_sync(0xffffffffu, TR, 31);
                if (m <= n) {
                    bad |= !(TR < dmin[m]);
                    if (m == n) bad |= TR > tbt_bound;
                    if (trow) trow[m - 1] = TR;
                }
            }
            if (__any_sync(0xffffffffu, bad)) {
                ok = false;
                if (!trow) break;
            }
        }
        if (lane == 0) {
            s_pass[u] = ok;
            if (ok) atomicMin(&s_best, u);
        }
    }
    __syncthreads();
    finish(i, F, st, 0u, s_pass, level, status);
}

struct WsView {
    const int32_t* run_h;
    const int32_t* run_m;
    const uint32_t* run_key;
    const int32_t* cell_tab;
    const float* lut;
    const uint32_t* cell_clamp;
};

// One warp: does level u pass?  T_R is formed run by run from the LUT (exact ticks) and checked at
// the compacted end positions (e_l, e_d) and, for the TBT check, at m = n.  Without trow the scan
// stops at the first violated deadline; with trow every T_R[m] of the level is written.
__device__ __forceinline__ bool level_passes_runs(const WsView& ws, int F, int u, int h, int ne,
                                                  const int* r_start, const int* r_row, const int* e_l,
                                                  const long long* e_d, long long tbt_bound, long long* trow) {
    const int lane = threadIdx.x & 31;
    long long carry = 0;     // T_R at the last iteration before the current chunk of runs
    int ep = 0;              // next end position to check
    bool ok = true;
    for (int kb = 0; kb < h; kb += 32) {
        const int k = kb + lane;
        int s = 0x7fffffff;
        long long t = 0, own = 0;
        if (k < h) {
            s = r_start[k];
            t = ticks_of(__ldg(ws.lut + (size_t)r_row[k] * F + u));
            own = (long long)(r_start[k + 1] - s) * t;      // the run's share of T_R, exact
        }
        long long x = own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const long long before = carry + x - own;           // T_R at iteration s - 1
        const int chunk_end = r_start[min(kb + 32, h)] - 1;  // last iteration of this chunk
        bool bad = false;
        // end positions inside this chunk: lane j checks e_l[ep + j]
        while (ep < ne && e_l[ep] <= chunk_end) {
            const int j = ep + lane;
            const int e = (j < ne) ? e_l[j] : 0x7fffffff;
            const bool mine = e <= chunk_end;
            int r = 0;   // last run of the chunk with start <= e
#pragma unroll
            for (int step = 16; step; step >>= 1) {
                const int cand = r + step;
                const int sc = __shfl_sync(0xffffffffu, s, cand);
                if (sc <= e) r = cand;
            }
            const long long b = __shfl_sync(0xffffffffu, before, r);
            const long long tt = __shfl_sync(0xffffffffu, t, r);
            const int sr = __shfl_sync(0xffffffffu, s, r);
            if (mine) bad |= !(b + (long long)(e - sr + 1) * tt < e_d[j]);
            ep += __popc(__ballot_sync(0xffffffffu, mine));
        }
        if (trow && k < h)
            for (int m = s; m < r_start[k + 1]; ++m) trow[m - 1] = before + (long long)(m - s + 1) * t;
        carry = __shfl_sync(0xffffffffu, carry + x, 31);
        if (__any_sync(0xffffffffu, bad)) {
            ok = false;
            if (!trow) break;
        }
    }
    return ok && carry <= tbt_bound;          // TBT at m = n: T_R[n] <= n * slo
}

// SEARCH = 0: exhaustive (reading A-13): levels strided over the warps, a warp skips levels above
//             one that already passed.
// SEARCH = 1: the paper's binary search (reading A-24), speculatively unrolled: each
//             round evaluates, one warp per level, the next levels of the search tree from the
//             current [lo, hi] (the top level F-1 first, then the mids of the first 3 bisection
//             steps: 1 + 2 + 4 nodes), then walks the path the sequential search takes.  Only the
//             path's levels count (IPS_CLAMPED included); F = 32 takes 2 rounds, 11 evaluations.
template <int SEARCH>
__global__ void __launch_bounds__(kThreads)
k3_select_runs(const tp_inst* __restrict__ inst, const int4* __restrict__ req, const double* __restrict__ t_dead,
               const int32_t* __restrict__ nv, const int32_t* __restrict__ nadm, int32_t H, int32_t F,
               long long tbt_ticks, int32_t* __restrict__ level, uint32_t* __restrict__ status,
               long long* __restrict__ tr, const __grid_constant__ WsView ws) {
    // shared: dmin[n + 1] (int64) | e_d[n] (int64) | e_l[n] | r_start[h + 1] | r_row[h]
    extern __shared__ long long sm[];
    __shared__ int s_pass[kMaxF];
    __shared__ int s_best;
    __shared__ int swarp[kWarps], swarp_ex[kWarps + 1];
    const int i = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t st = status[i];
    if (st & kSkip) {
        if (tid == 0) level[i] = (st & TP_ST_BAD_INPUT) ? F - 1 : (st & TP_ST_EMPTY) ? 0 : F - 1;
        return;
    }
    const int n = nv[i];
    const size_t row = (size_t)i * H;
    const int h = ws.run_h[i];
    long long* dmin = sm;
    long long* e_d = dmin + (n + 1);
    int* e_l = reinterpret_cast<int*>(e_d + n);
    int* r_start = e_l + n;
    int* r_row = r_start + (h + 1);
    const tp_inst in = inst[i];
    if (tid < kMaxF) s_pass[tid] = 0;
    if (tid == 0) s_best = F;
    // runs: first iteration and LUT row; clamp mask from the cells' masks
    uint32_t cl = 0;
    for (int k = tid; k < h; k += kThreads) {
        r_start[k] = __ldg(ws.run_m + row + k);
        const uint32_t key = __ldg(ws.run_key + row + k);
        r_row[k] = __ldg(ws.cell_tab + key);
        cl |= __ldg(ws.cell_clamp + key);
    }
    if (tid == 0) r_start[h] = n + 1;
    for (int o = 16; o; o >>= 1) cl |= __shfl_xor_sync(0xffffffffu, cl, o);
    if (lane == 0) swarp[warp] = (int)cl;
    __syncthreads();
    uint32_t clamp_mask = 0;     // bit u: some value of level u was clamped
    for (int w = 0; w < kWarps; ++w) clamp_mask |= (uint32_t)swarp[w];
    build_dmin(dmin, in, in.n_run + nadm[i], n, req, t_dead);
    // compact the end positions that carry a deadline (ascending)
    int ne = 0;
    for (int m0 = 1; m0 <= n; m0 += kThreads) {
        const int m = m0 + tid;
        const bool has = m <= n && dmin[m] != kNoDeadline;
        const unsigned mask = __ballot_sync(0xffffffffu, has);
        if (lane == 0) swarp[warp] = __popc(mask);
        __syncthreads();
        if (tid < 32) {      // exclusive scan of the warp counts (one warp)
            const int c = lane < kWarps ? swarp[lane] : 0;
            int x = c;
#pragma unroll
            for (int o = 1; o < kWarps; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane < kWarps) swarp_ex[lane] = x - c;
            if (lane == kWarps - 1) swarp_ex[kWarps] = x;
        }
        __syncthreads();
        const int before = ne + swarp_ex[warp];
        if (has) {
            const int pos = before + __popc(mask & ((1u << lane) - 1u));
            e_l[pos] = m;
            e_d[pos] = dmin[m];
        }
        ne += swarp_ex[kWarps];
        __syncthreads();
    }

    const long long tbt_bound = (long long)n * tbt_ticks;
    if constexpr (SEARCH == 0) {
        for (int u = warp; u < F; u += kWarps) {
            if (!tr && u > *(volatile int*)&s_best) break;      // a lower level already passed
            long long* trow = tr ? tr + ((size_t)i * F + u) * H : nullptr;
            const bool ok = level_passes_runs(ws, F, u, h, ne, r_start, r_row, e_l, e_d, tbt_bound, trow);
            if (lane == 0) {
                s_pass[u] = ok;
                if (ok) atomicMin(&s_best, u);
            }
        }
        __syncthreads();
        finish(i, F, st, clamp_mask ? (uint32_t)TP_ST_IPS_CLAMPED : 0u, s_pass, level, status);
    } else {
        __shared__ int s_lv[kWarps], s_ok[kWarps];
        __shared__ int s_nlv, s_lo, s_hi, s_state;   // state 0: top level pending, 1: bisecting, 2: done, 3: infeasible
        __shared__ uint32_t s_vis;
        if (tid == 0) {
            s_lo = 0;
            s_hi = F - 1;
            s_state = 0;
            s_vis = 0;
        }
        __syncthreads();
        while (true) {
            if (tid == 0) {          // plan: breadth-first over the bisection tree from [lo, hi]
                int k = 0;
                if (s_state == 0) s_lv[k++] = F - 1;
                int qlo[16], qhi[16], qh = 0, qt = 0;
                qlo[qt] = s_lo;
                qhi[qt++] = s_hi;
                while (qh < qt && k < kWarps) {
                    const int lo = qlo[qh], hi = qhi[qh++];
                    if (lo >= hi) continue;
                    const int mid = (lo + hi) >> 1;
                    s_lv[k++] = mid;
                    if (qt + 2 <= 16) {
                        qlo[qt] = lo; qhi[qt++] = mid;          // pass(mid) -> [lo, mid]
                        qlo[qt] = mid + 1; qhi[qt++] = hi;      // fail      -> [mid + 1, hi]
                    }
                }
                s_nlv = k;
            }
            __syncthreads();
            if (warp < s_nlv) {
                const bool ok = level_passes_runs(ws, F, s_lv[warp], h, ne, r_start, r_row, e_l, e_d, tbt_bound,
                                                  nullptr);
                if (lane == 0) s_ok[warp] = ok;
            }
            __syncthreads();
            if (tid == 0) {          // walk the path the sequential search takes
                int k0 = 0;
                if (s_state == 0) {
                    s_vis |= 1u << (F - 1);
                    s_state = s_ok[0] ? 1 : 3;
                    k0 = 1;
                }
                if (s_state == 1) {
                    int lo = s_lo, hi = s_hi;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        int j = -1;
                        for (int q = k0; q < s_nlv; ++q)
                            if (s_lv[q] == mid) j = q;
                        if (j < 0) break;    // beyond this round's plan
                        s_vis |= 1u << mid;
                        if (s_ok[j]) hi = mid;
                        else lo = mid + 1;
                    }
                    s_lo = lo;
                    s_hi = hi;
                    if (lo >= hi) s_state = 2;
                }
            }
            __syncthreads();
            if (s_state >= 2) break;
        }
        if (tid == 0) {
            const uint32_t st_or = (clamp_mask & s_vis) ? (uint32_t)TP_ST_IPS_CLAMPED : 0u;
            if (s_state == 2) {
                level[i] = s_lo;
                if (st_or) status[i] = st | st_or;
            } else {
                level[i] = F - 1;
                status[i] = st | st_or | TP_ST_INFEASIBLE;
            }
        }
    }
}

bool set_attr(const void* fn, int bytes, bool* done, int dev) {
    if (dev < 64 && done[dev]) return true;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
    if (dev < 64) done[dev] = true;
    return true;
}

}  // namespace

int launch_select(const tp_inst* inst, int32_t n_inst, const tp_req* req, int32_t n_req, const double* t_dead,
                  const int32_t* n, const int32_t* n_adm, const float* ips, int32_t H, int32_t F,
                  int64_t tbt_ticks, int32_t* level, uint32_t* status, int64_t* tr, const K2Params* ws,
                  int search, cudaStream_t s) {
    (void)n_req;
    if (n_inst == 0) return TP_OK;
    if (search != 0 && (search != 1 || !ws)) return TP_EINVAL;   // binary search: LUT path only
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return TP_ECUDA;
    if (!ws) {
        static bool done[64] = {};
        if (!set_attr((const void*)k3_select, (kMaxH + 1) * 8, done, dev)) return TP_ECUDA;
        k3_select<<<n_inst, kThreads, (size_t)(H + 1) * 8, s>>>(inst, reinterpret_cast<const int4*>(req), t_dead, n,
                                                                n_adm, ips, H, F, (long long)tbt_ticks, level, status,
                                                                reinterpret_cast<long long*>(tr));
    } else {
        // dmin (H+1) + e_d H (int64) + e_l H + r_start (H+1) + r_row H (int32)
        auto bytes = [](size_t h) { return (h + 1) * 8 + h * 8 + h * 4 + (h + 1) * 4 + h * 4; };
        if (H > kMaxHRunsSelect || (search == 1 && tr)) return TP_EINVAL;
        auto kern = search == 1 ? k3_select_runs<1> : k3_select_runs<0>;
        static bool done[2][64] = {};
        if (!set_attr((const void*)kern, (int)bytes(kMaxHRunsSelect), done[search == 1], dev)) return TP_ECUDA;
        WsView v{ws->run_h, ws->run_m, ws->run_key, ws->cell_tab, ws->lut, ws->cell_clamp};
        kern<<<n_inst, kThreads, bytes((size_t)H), s>>>(inst, reinterpret_cast<const int4*>(req), t_dead, n, n_adm, H,
                                                        F, (long long)tbt_ticks, level, status,
                                                        reinterpret_cast<long long*>(tr), v);
    }
    return cudaPeekAtLastError() == cudaSuccess ? TP_OK : TP_ECUDA;
}

}  // namespace tp
