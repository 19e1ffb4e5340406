// K3 -- SLO scan and frequency choice: T' = 1/IPS, T_R = cumulative sum (Eq. 3),
// TBT check, E2E check Eq. 4, lowest SLO-meeting frequency with
// the lost bypass.
//
// One CTA per instance, one warp per frequency level (levels strided over the 8 warps).
//  * Per instance, the scheduled requests' deadlines become a table Dmin[l] = min over requests
//    ending at l of ceil(fl64(t_dead - t_cur) * 2^40) (int64 ticks of 2^-40 s) in shared memory,
//    so Eq. 4 for every request is "T_R[m] < Dmin[m] for all m <= n".
//  * T'[m] = fl32(1/ips) lies in [2^-17, 16] s, i.e. an integer number of 2^-40 s ticks, so the
//    warp computes the cumulative sum exactly with an int64 shuffle scan (reading A-10): any
//    summation order gives the same bits, and the SLO comparisons are exact integer compares.
//  * A warp stops scanning at the first violated deadline (unless T_R is requested).
//  * The decision is the lowest passing level: a ballot over the per-level pass flags.
#include "tp_internal.cuh"

namespace tp {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kSkip = TP_ST_BAD_INPUT | TP_ST_EMPTY | TP_ST_BYPASS_LOST;

// ceil(s * 2^40) for the E2E compare T_R < s (T_R integer ticks): <= 0 / NaN -> 0 (never passes),
// >= 2^62 -> INT64_MAX (always passes; T_R < 2^58).
__device__ __forceinline__ long long slack_ticks(double s) {
    const double d = s * 0x1p40;
    if (!(d > 0.0)) return 0;
    if (d >= 0x1p62) return 0x7fffffffffffffffLL;
    return (long long)ceil(d);
}

// WS = false: IPS read from the ips grid.  WS = true (fused with K2's cell mode): IPS read from the
// cell LUT through the instance's runs, so the ips grid is never materialised.
struct WsView {
    const int32_t* run_h;
    const int32_t* run_m;
    const uint32_t* run_key;
    const int32_t* cell_tab;
    const float* lut;
    const uint32_t* cell_clamp;
};

template <bool WS>
__global__ void __launch_bounds__(kThreads)
k3_select(const tp_inst* __restrict__ inst, const int4* __restrict__ req, const double* __restrict__ t_dead,
          const int32_t* __restrict__ nv, const int32_t* __restrict__ nadm, const float* __restrict__ ips,
          int32_t H, int32_t F, long long tbt_ticks, int32_t* __restrict__ level, uint32_t* __restrict__ status,
          long long* __restrict__ tr, const __grid_constant__ WsView ws) {
    extern __shared__ long long dmin[];   // index m in [1, n]; (WS) then int lrow[m], m in [1, n]
    __shared__ int s_pass[kMaxF];
    const int i = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t st = status[i];
    if (st & kSkip) {
        if (tid == 0) level[i] = (st & TP_ST_BAD_INPUT) ? F - 1 : (st & TP_ST_EMPTY) ? 0 : F - 1;
        return;
    }
    const int n = nv[i];
    const tp_inst in = inst[i];
    for (int m = tid; m <= n; m += kThreads) dmin[m] = 0x7fffffffffffffffLL;
    int* lrow = reinterpret_cast<int*>(dmin + (n + 1));
    uint32_t st_or = 0;
    if constexpr (WS) {
        // LUT row of every iteration: its run's cell (binary search over the run starts)
        const size_t row = (size_t)i * H;
        const int h = ws.run_h[i];
        for (int m = 1 + tid; m <= n; m += kThreads) {
            int lo = 0, hi = h;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (__ldg(ws.run_m + row + mid) <= m) lo = mid;
                else hi = mid;
            }
            lrow[m] = __ldg(ws.cell_tab + __ldg(ws.run_key + row + lo));
        }
        bool cl = false;
        for (int k = tid; k < h; k += kThreads) cl |= __ldg(ws.cell_clamp + __ldg(ws.cell_tab + __ldg(ws.run_key + row + k))) != 0;
        if (__syncthreads_or(cl)) st_or = TP_ST_IPS_CLAMPED;
    }
    __syncthreads();
    const int nsched = in.n_run + nadm[i];
    for (int e = tid; e < nsched; e += kThreads) {
        const int64_t j = (int64_t)in.req_begin + e;
        const int4 r = __ldg(&req[j]);
        const double slack = __ldg(&t_dead[j]) - in.t_cur;   // fl64(t_dead - t_cur), reading A-12
        atomicMin(&dmin[r.z - r.x], slack_ticks(slack));
    }
    __syncthreads();

    const long long tbt_bound = (long long)n * tbt_ticks;   // TBT: T_R[n] <= n * slo (<= 2^58)
    for (int u = warp; u < F; u += kWarps) {
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
                if constexpr (WS) v[j] = m <= n ? __ldg(ws.lut + (size_t)lrow[m] * F + u) : 1.0f;
                else v[j] = m <= n ? __ldg(row + m - 1) : 1.0f;
            }
            bool bad = false;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int m = m0 + 32 * j + lane;
                long long x = 0;
                if (m <= n) {
                    const float t = __frcp_rn(v[j]);                   // fl32(1 / IPS), reading A-9
                    x = (long long)(t * 0x1p40f);                      // exact: t in [2^-17, 16]
                }
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
        if (lane == 0) s_pass[u] = ok;
    }
    __syncthreads();
    if (warp == 0) {
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
}

}  // namespace

int launch_select(const tp_inst* inst, int32_t n_inst, const tp_req* req, int32_t n_req, const double* t_dead,
                  const int32_t* n, const int32_t* n_adm, const float* ips, int32_t H, int32_t F,
                  int64_t tbt_ticks, int32_t* level, uint32_t* status, int64_t* tr, const K2Params* ws,
                  cudaStream_t s) {
    (void)n_req;
    if (n_inst == 0) return TP_OK;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return TP_ECUDA;
    static bool attr_done[2][64] = {};
    WsView v{};
    if (ws) {
        v.run_h = ws->run_h;
        v.run_m = ws->run_m;
        v.run_key = ws->run_key;
        v.cell_tab = ws->cell_tab;
        v.lut = ws->lut;
        v.cell_clamp = ws->cell_clamp;
    }
    const size_t smem = (size_t)(H + 1) * (sizeof(long long) + (ws ? 4 : 0));
    const void* fn = ws ? (const void*)k3_select<true> : (const void*)k3_select<false>;
    if (dev < 64 && !attr_done[ws ? 1 : 0][dev]) {
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (kMaxH + 1) * 12) != cudaSuccess)
            return TP_ECUDA;
        attr_done[ws ? 1 : 0][dev] = true;
    }
    if (ws)
        k3_select<true><<<n_inst, kThreads, smem, s>>>(inst, reinterpret_cast<const int4*>(req), t_dead, n, n_adm,
                                                       nullptr, H, F, (long long)tbt_ticks, level, status,
                                                       reinterpret_cast<long long*>(tr), v);
    else
        k3_select<false><<<n_inst, kThreads, smem, s>>>(inst, reinterpret_cast<const int4*>(req), t_dead, n, n_adm,
                                                        ips, H, F, (long long)tbt_ticks, level, status,
                                                        reinterpret_cast<long long*>(tr), v);
    return cudaPeekAtLastError() == cudaSuccess ? TP_OK : TP_ECUDA;
}

}  // namespace tp
