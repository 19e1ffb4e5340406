// K3c -- the compact path's SLO scan and frequency choice: T' = 1/IPS (reading A-9),
// T_R = cumulative sum (Eq. 3, exact int64 ticks, reading A-10), TBT check, E2E
// check Eq. 4 and the lowest SLO-meeting frequency.
//
// One WARP per instance, lane u = frequency level u (F <= 32): every lane walks the same sequence
// of runs (from K1c) and end positions (K1c's deadline list) in m order -- the control flow is
// warp-uniform, only the IPS value differs per lane -- so
//   * on a run [s, s') with constant T' = t (its cell's row of K2's tick LUT, one coalesced load for
//     all levels), T_R grows by (s' - s) * t, exactly;
//   * an end position l inside the run checks T_R[s-1] + (l - s + 1) * t < Dmin[l] (strict, Eq. 4);
//   * the TBT check is T_R[n] <= n * tbt_slo (tie passes);
// and the decision is one __ballot_sync over the levels' pass bits: __ffs of it (exhaustive,
// reading A-13) or the paper's binary search replayed on the bit vector (reading A-24; the search
// visits F-1 first, then the mids).  IPS_CLAMPED: the OR of the cells' clamp masks over the runs,
// restricted to the visited levels (all F in the exhaustive order).
#include <cstdlib>

#include "tp_internal.cuh"

namespace tp {
namespace {

constexpr int kWarpsPerCta = 8;
constexpr unsigned kFull = 0xffffffffu;
// W = 1 (large batches, throughput): 8 CTAs per SM and 2 LUT rows prefetched; W > 1 (small
// batches, latency): 4 CTAs per SM, 8 rows prefetched and the next run chunk loaded ahead
// (measured on C3 / C2)
#ifndef TP_K3C_PREFETCH
#define TP_K3C_PREFETCH 2
#endif
#ifndef TP_K3C_MINB
#define TP_K3C_MINB 8
#endif      // LUT values loaded ahead per lane

// TP_K3C_WARPS (1/2/4/8): warps per instance override (tuning)
int env_warps() {
    const char* v = std::getenv("TP_K3C_WARPS");
    const int x = v ? std::atoi(v) : 0;
    return (x == 1 || x == 2 || x == 4 || x == 8) ? x : 0;
}

struct K3cParams {
    const int32_t* n;
    uint32_t* status;
    int32_t* level;
    const int32_t* run_h;
    const int32_t* run_m;
    const uint32_t* run_key;
    const int32_t* cell_tab;
    const long long* lut_ticks;
    const uint32_t* cell_clamp;
    const int32_t* end_n;
    const int32_t* end_l;
    const long long* end_d;
    int32_t n_inst, H, F;
    long long tbt_ticks;
    uint32_t skip;
    int32_t search;
};

// #entries of the ascending array a[0, cnt) that are < x, by the whole warp (32-way sampling:
// one dependent load per factor 32 of cnt).
__device__ __forceinline__ int warp_lower_bound(const int* __restrict__ a, int cnt, int x) {
    const int lane = threadIdx.x & 31;
    int lo = 0, len = cnt;                       // answer in [lo, lo + len]
    while (len > 32) {
        const int stride = (len + 31) / 32;
        const int k = lo + lane * stride;
        const bool lt = k < lo + len && __ldg(a + k) < x;
        const int c = __popc(__ballot_sync(kFull, lt));    // samples < x (a prefix of the lanes)
        if (c == 0) return lo;
        lo += (c - 1) * stride + 1;
        len = min(stride - 1, cnt - lo);
    }
    const bool lt = lane < len && __ldg(a + lo + lane) < x;
    return lo + __popc(__ballot_sync(kFull, lt));
}

// W warps per instance: warp w walks the runs [h*w/W, h*(w+1)/W) and the end positions inside
// them with a local T_R starting at 0; it leaves its total S_w[u] and its Eq. 4 margin
// M_w[u] = min over its ends of (Dmin[l] - T_local(l)) (integers, exact); the instance passes at u
// iff P_w < M_w for every w, P_w = S_0 + ... + S_{w-1} (T_R[l] = P_w + T_local(l) < Dmin[l]), and
// the TBT check holds on the total.  W = 1 keeps the early exit once every level has failed.
template <int W>
__global__ void __launch_bounds__(kWarpsPerCta * 32, W == 1 ? TP_K3C_MINB : 4)
k3_compact(const __grid_constant__ K3cParams p) {
    constexpr int IPC = kWarpsPerCta / W;            // instances per CTA
    __shared__ long long s_S[W > 1 ? kWarpsPerCta : 1][32], s_M[W > 1 ? kWarpsPerCta : 1][32];
    __shared__ uint32_t s_cm[W > 1 ? kWarpsPerCta : 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = warp / W, w = warp % W;             // instance slot in the CTA, segment
    const int i = blockIdx.x * IPC + g;
    const bool live = i < p.n_inst;
    pdl_wait();                                       // K1c / K2 outputs
    const int F = p.F;
    uint32_t st = 0;
    bool skipped = true;
    if (live) {
        st = p.status[i];
        skipped = (st & p.skip) != 0;
        if (skipped && w == 0 && lane == 0)
            p.level[i] = (st & TP_ST_BAD_INPUT) ? F - 1 : (st & TP_ST_EMPTY) ? 0 : F - 1;
    }
    if (W == 1 && (!live || skipped)) return;
    const bool work = live && !skipped;               // warp-uniform (same instance for the W warps)
    const bool act = lane < F;
    long long T = 0;                                  // local T_R before the current run
    long long M = kNoDeadline;                        // Eq. 4 margin (W > 1)
    bool ok = act;                                    // W == 1: pass so far
    uint32_t cm = 0;                                  // OR of the runs' cell clamp masks
    int n = 0;
    if (work) {
        n = p.n[i];
        const int h = p.run_h[i], ne = p.end_n[i];
        const size_t row = (size_t)i * p.H;
        const int ka = (int)((int64_t)h * w / W), kz = (int)((int64_t)h * (w + 1) / W);
        int ea = 0, ez = ne;
        if (W > 1) {
            const int sa = ka < h ? __ldg(p.run_m + row + ka) : n + 1;
            const int sz = kz < h ? __ldg(p.run_m + row + kz) : n + 1;
            ea = w == 0 ? 0 : warp_lower_bound(p.end_l + row, ne, sa);
            ez = w == W - 1 ? ne : warp_lower_bound(p.end_l + row, ne, sz);
        }
        // end positions of this segment, 32 per chunk in registers; the current one by shuffle
        int eb = ea;
        int el = (eb + lane < ez) ? __ldg(p.end_l + row + eb + lane) : 0x7fffffff;
        long long ed = (eb + lane < ez) ? __ldg(p.end_d + row + eb + lane) : 0;
        int ep = ea;
        int cur_l = __shfl_sync(kFull, el, 0);        // INT_MAX when the segment has no end
        long long cur_d = __shfl_sync(kFull, ed, 0);
        // this level's column of the tick LUT (W = 1: lanes >= F read column F-1 -- in the row,
        // ignored -- instead of a predicated load; fewer live registers)
        const int lc = W == 1 ? min(lane, F - 1) : lane;
        // run chunk kb: start, length and LUT row per lane; the next chunk's records are loaded
        // while the current one is walked
        int nx_s = n + 1, nx_len = 0;
        uint32_t nx_key = 0;
        auto load_chunk = [&](int kb) {
            const int k = kb + lane;
            nx_s = n + 1;
            nx_len = 0;
            nx_key = 0;
            if (k < kz) {
                nx_s = __ldg(p.run_m + row + k);
                nx_len = ((k + 1 < h) ? __ldg(p.run_m + row + k + 1) : n + 1) - nx_s;
                nx_key = __ldg(p.run_key + row + k);
            }
        };
        // W = 1 (large batches, 8 CTAs/SM at 32 registers): no look-ahead load -- the registers it
        // needs cost more in spills than it saves in latency (C3: 535 -> 505 us with 2-row prefetch)
        constexpr bool kNext = W > 1;
        if constexpr (kNext) load_chunk(ka);
        for (int kb = ka; kb < kz; kb += 32) {
            if constexpr (!kNext) load_chunk(kb);
            const int s_k = nx_s, len_k = nx_len;
            const int rr = (kb + lane < kz) ? __ldcg(p.cell_tab + nx_key) : 0;
            const int roff = rr * F;                  // the run's LUT row offset (< 2^27)
            if constexpr (kNext)
                if (kb + 32 < kz) load_chunk(kb + 32);
            if (kb + lane < kz) cm |= __ldcg(p.cell_clamp + rr);
            const int cnt = min(32, kz - kb);
            constexpr int kPrefetch = W == 1 ? TP_K3C_PREFETCH : 8;
            for (int j0 = 0; j0 < cnt; j0 += kPrefetch) {
                long long tv[kPrefetch];
#pragma unroll
                for (int q = 0; q < kPrefetch; ++q) {
                    const int o_ = __shfl_sync(kFull, roff, (j0 + q) & 31);
                    tv[q] = (W == 1 || act) ? __ldcg(p.lut_ticks + (unsigned)(o_ + lc)) : 0;   // rows past cnt: row 0
                }
#pragma unroll
                for (int q = 0; q < kPrefetch; ++q) {
                    if (j0 + q < cnt) {                  // uniform
                        const int s = __shfl_sync(kFull, s_k, j0 + q), len = __shfl_sync(kFull, len_k, j0 + q);
                        const long long t = tv[q];
                        const long long Tm = T - (long long)(s - 1) * t;   // T_R(l) = Tm + l * t on the run
                        while (cur_l < s + len) {        // end positions inside this run (>= s: sorted)
                            const long long tl = Tm + (long long)cur_l * t;
                            if (W == 1) ok &= tl < cur_d;
                            else M = min(M, cur_d - tl);
                            if (++ep - eb == 32) {
                                eb += 32;
                                el = (eb + lane < ez) ? __ldg(p.end_l + row + eb + lane) : 0x7fffffff;
                                ed = (eb + lane < ez) ? __ldg(p.end_d + row + eb + lane) : 0;
                            }
                            cur_l = __shfl_sync(kFull, el, ep - eb);
                            cur_d = __shfl_sync(kFull, ed, ep - eb);
                        }
                        T += (long long)len * t;
                    }
                }
            }
            if (W == 1 && !__any_sync(kFull, ok)) {      // every level failed: only the clamp OR is left
                for (int k2 = kb + 32 + lane; k2 < kz; k2 += 32)
                    cm |= __ldcg(p.cell_clamp + __ldcg(p.cell_tab + __ldg(p.run_key + row + k2)));
                break;
            }
        }
    }
    cm = __reduce_or_sync(kFull, cm);
    if (W > 1) {
        s_S[warp][lane] = T;
        s_M[warp][lane] = M;
        if (lane == 0) s_cm[warp] = cm;
        __syncthreads();
        if (w != 0 || !work) return;
        long long P = 0;
#pragma unroll
        for (int v = 0; v < W; ++v) {
            ok &= P < s_M[g * W + v][lane];
            P += s_S[g * W + v][lane];
            cm |= s_cm[g * W + v];
        }
        T = P;
    }
    ok &= T <= (long long)n * p.tbt_ticks;           // TBT: T_R[n] <= n * slo
    const uint32_t pass = __ballot_sync(kFull, ok);
    if (lane == 0) {
        const uint32_t fmask = F == 32 ? 0xffffffffu : ((1u << F) - 1u);
        uint32_t vis, out = st;
        int lv;
        if (p.search == 0) {
            vis = fmask;
            lv = pass ? __ffs(pass) - 1 : F - 1;
            if (!pass) out |= TP_ST_INFEASIBLE;
        } else {
            vis = 1u << (F - 1);
            if (!((pass >> (F - 1)) & 1u)) {
                lv = F - 1;
                out |= TP_ST_INFEASIBLE;
            } else {
                int lo = 0, hi = F - 1;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    vis |= 1u << mid;
                    if ((pass >> mid) & 1u) hi = mid;
                    else lo = mid + 1;
                }
                lv = lo;
            }
        }
        if (cm & vis) out |= TP_ST_IPS_CLAMPED;
        p.level[i] = lv;
        if (out != st) p.status[i] = out;
    }
}

}  // namespace

int launch_select_compact(const K2Params& w, int32_t n_inst, const int32_t* n, int32_t H, int32_t F,
                          int64_t tbt_ticks, int search, uint32_t skip, int32_t* level, uint32_t* status,
                          cudaStream_t s) {
    if (n_inst == 0) return TP_OK;
    if (!w.cell_tab || !w.end_n || F < 1 || F > kMaxF || (search != 0 && search != 1)) return TP_EINVAL;
    K3cParams p;
    p.n = n;
    p.status = status;
    p.level = level;
    p.run_h = w.run_h;
    p.run_m = w.run_m;
    p.run_key = w.run_key;
    p.cell_tab = w.cell_tab;
    p.lut_ticks = w.lut_ticks;
    p.cell_clamp = w.cell_clamp;
    p.end_n = w.end_n;
    p.end_l = w.end_l;
    p.end_d = w.end_d;
    p.n_inst = n_inst;
    p.H = H;
    p.F = F;
    p.tbt_ticks = (long long)tbt_ticks;
    p.skip = skip;
    p.search = search;
    // warps per instance: enough warps to fill the GPU at small batches (the walk of one instance is
    // a dependent chain of L2 round trips), one per instance at large ones
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static const int w_env = env_warps();
    const int64_t slots = (int64_t)sms * 32;          // resident warps at 8-warp CTAs, 4 per SM
    int W = w_env > 0 ? w_env : (n_inst * 8 <= slots ? 8 : n_inst * 4 <= slots ? 4 : n_inst * 2 <= slots ? 2 : 1);
    auto launch = [&](auto kern, int ipc) {
        const int grid = (n_inst + ipc - 1) / ipc;
        launch_pdl(kern, dim3(grid), dim3(kWarpsPerCta * 32), 0, s, p);
    };
    switch (W) {
        case 8: launch(k3_compact<8>, 1); break;
        case 4: launch(k3_compact<4>, 2); break;
        case 2: launch(k3_compact<2>, 4); break;
        default: launch(k3_compact<1>, 8); break;
    }
    return cudaPeekAtLastError() == cudaSuccess ? TP_OK : TP_ECUDA;
}

}  // namespace tp
