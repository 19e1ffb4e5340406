// K2 -- the performance model M (PAPER §4.3.1) evaluated on the full
// (instance x frequency x future iteration) grid: ips = clamp(base + sum_t leaf_t(x)) with
// x = (tp, B[m], KV[m], f_u), leaves added in fp32 in tree order (reading A-7).
//
// Design (sm_100a):
//  * A warp owns a tile = 32 consecutive iterations m of one instance x RU frequency levels; each
//    lane evaluates RU grid rows (same m, RU frequencies) -> RU independent descents for ILP.
//  * Features are replaced by their ranks among the ensemble's sorted distinct thresholds
//    (rank = #cuts <= x; x < cut_j <=> rank <= j), packed 16 bits each into two registers.
//  * Trees are complete heaps of 32-bit words staged in shared memory by TMA (cp.async.bulk,
//    mbarrier completion), double-buffered in chunks when the model exceeds the smem budget;
//    every CTA streams the chunks in the same fixed order, so the per-row fp32 sums are formed in
//    tree order.
//  * One tree level costs 4 instructions per row: LDS (word), PRMT (pick the split feature's rank
//    into the upper half), IADD3 with carry-out (rank + 0xFFFF - j overflows <=> go right) and
//    IADD3.X (idx = 2*idx + carry).  No branches, no divergence.
//  * Persistent-style grid (#SMs x occupancy CTAs); tiles are split evenly over CTAs by a
//    per-CTA scan of the per-instance tile counts.
#include <algorithm>

#include "tp_internal.cuh"

namespace tp {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunkBytes = 48 * 1024;
constexpr uint32_t kSkip = TP_ST_BAD_INPUT | TP_ST_EMPTY | TP_ST_BYPASS_LOST;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    uint32_t polls = 0;
    do {
        if (++polls == (1u << 28)) __trap();   // a lost TMA completion must fail, never hang the GPU
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// One tree level: idx' = 2*idx + go_right, go_right = carry_out(prmt(xlo, xhi, w) + w).
__device__ __forceinline__ uint32_t descend(uint32_t idx, uint32_t w, uint32_t xlo, uint32_t xhi) {
    uint32_t out;
    asm("{\n\t.reg .b32 pr, t;\n\t"
        "prmt.b32 pr, %1, %2, %3;\n\t"
        "add.cc.u32 t, pr, %3;\n\t"
        "addc.u32 %0, %4, %4;\n\t}"
        : "=r"(out)
        : "r"(xlo), "r"(xhi), "r"(w), "r"(idx));
    return out;
}

__device__ __forceinline__ uint32_t rank_of(const float* __restrict__ c, int cnt, float x) {
    int lo = 0, hi = cnt;   // upper bound: number of cuts <= x
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(c + mid) <= x) lo = mid + 1;
        else hi = mid;
    }
    return (uint32_t)lo;
}

__device__ __forceinline__ int64_t tiles_of(const int32_t* __restrict__ n, const uint32_t* __restrict__ st,
                                            int i, int G) {
    return (st[i] & kSkip) ? 0 : (int64_t)((n[i] + 31) >> 5) * G;
}

template <int D, int RU>
__global__ void __launch_bounds__(kThreads, 2)
k2_gbdt(const __grid_constant__ K2Params p, int TC, int nchunks) {
    extern __shared__ __align__(128) uint32_t sw[];
    __shared__ __align__(8) uint64_t full[2];
    __shared__ int64_t red[kWarps];
    __shared__ int64_t s_start_pc;
    __shared__ int s_start_i;
    __shared__ uint32_t s_rf[kMaxF];

    constexpr int TW = (2 << D) < 4 ? 4 : (2 << D);    // words per tree (>= 16 B for TMA)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = (p.F + RU - 1) / RU;
    const int I = p.n_inst;
    const bool resident = nchunks == 1;
    const int stages = resident ? 1 : 2;
    const int chunk_words = TC * TW;

    if (tid < p.F)
        s_rf[tid] = rank_of(p.cuts + p.cut_off[3], p.cut_off[4] - p.cut_off[3], p.freq[tid]);

    // ---- split the tile space [0, Ttot) evenly over CTAs ----
    int64_t tot = 0;
    for (int i = tid; i < I; i += kThreads) tot += tiles_of(p.n, p.status, i, G);
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0) red[warp] = tot;
    __syncthreads();
    tot = 0;
    for (int k = 0; k < kWarps; ++k) tot += red[k];
    const int64_t t0 = tot * blockIdx.x / gridDim.x, t1 = tot * (blockIdx.x + 1) / gridDim.x;
    if (t0 >= t1) return;   // uniform: no work for this CTA

    // locate the instance holding tile t0 (block-wide scan over instances, chunk by chunk)
    if (tid == 0) s_start_i = -1;
    __syncthreads();
    int64_t base_pc = 0;
    for (int c0 = 0; c0 < I; c0 += kThreads) {
        const int i = c0 + tid;
        const int64_t v = i < I ? tiles_of(p.n, p.status, i, G) : 0;
        int64_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        __syncthreads();
        if (lane == 31) red[warp] = x;
        __syncthreads();
        int64_t pre = base_pc;
        for (int k = 0; k < warp; ++k) pre += red[k];
        const int64_t incl = pre + x, excl = incl - v;
        if (i < I && v > 0 && excl <= t0 && t0 < incl) {
            s_start_i = i;
            s_start_pc = excl;
        }
        for (int k = 0; k < kWarps; ++k) base_pc += red[k];
        __syncthreads();
        if (s_start_i >= 0) break;
    }

    if (tid == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int nrounds = (int)((t1 - t0 + kWarps - 1) / kWarps);
    const int64_t total_loads = nchunks == 0 ? 0 : (resident ? 1 : (int64_t)nrounds * nchunks);
    auto issue = [&](int64_t g) {
        const int c = (int)(g % nchunks), s = (int)(g % stages);
        const int nt = min(TC, p.n_trees - c * TC);
        const uint32_t bytes = (uint32_t)nt * TW * 4u;
        mbar_expect_tx(&full[s], bytes);
        tma_load(sw + (size_t)s * chunk_words, p.words + (size_t)c * TC * TW, bytes, &full[s]);
    };
    if (tid == 0)
        for (int64_t g = 0; g < (total_loads < stages ? total_loads : (int64_t)stages); ++g) issue(g);

    int ci = s_start_i;        // per-warp cursor over instances (warp-uniform)
    int64_t pc = s_start_pc;   // tiles before instance ci
    int64_t g = 0;             // loads consumed so far
    const float* cutsB = p.cuts + p.cut_off[1];
    const float* cutsKV = p.cuts + p.cut_off[2];
    const float* cutsTP = p.cuts + p.cut_off[0];
    const int nB = p.cut_off[2] - p.cut_off[1], nKV = p.cut_off[3] - p.cut_off[2], nTP = p.cut_off[1] - p.cut_off[0];

    for (int round = 0; round < nrounds; ++round) {
        const int64_t t = t0 + (int64_t)round * kWarps + warp;
        const bool active = t < t1;
        int i = 0, m = 0, u0 = 0, ni = 0;
        uint32_t xlo = 0, xhi[RU];
        float acc[RU];
        if (active) {
            int64_t ti;
            while (t >= pc + (ti = tiles_of(p.n, p.status, ci, G)) && ci < I - 1) {
                pc += ti;
                ++ci;
            }
            i = ci;
            const int64_t tau = t - pc;
            const int mt = (int)(tau / G), ug = (int)(tau % G);
            ni = p.n[i];
            m = mt * 32 + lane + 1;
            u0 = ug * RU;
            const int tpv = p.inst[i].tp;
            int bv = 0, kvv = 0;
            if (m <= ni) {
                bv = p.B[(size_t)i * p.H + m - 1];
                kvv = p.KV[(size_t)i * p.H + m - 1];
            }
            xlo = rank_of(cutsTP, nTP, (float)tpv) | (rank_of(cutsB, nB, (float)bv) << 16);
            const uint32_t rkv = rank_of(cutsKV, nKV, (float)kvv);
#pragma unroll
            for (int r = 0; r < RU; ++r) xhi[r] = rkv | (s_rf[min(u0 + r, p.F - 1)] << 16);
        }
#pragma unroll
        for (int r = 0; r < RU; ++r) acc[r] = p.base;

        for (int c = 0; c < nchunks; ++c, ++g) {
            const int s = resident ? 0 : (int)(g % stages);
            mbar_wait(&full[s], resident ? 0u : (uint32_t)((g / stages) & 1));
            if (active) {
                const uint32_t* cw = sw + (size_t)s * chunk_words;
                const int nt = min(TC, p.n_trees - c * TC);
                for (int tt = 0; tt < nt; ++tt) {
                    const uint32_t* tw = cw + tt * TW;
                    uint32_t idx[RU];
#pragma unroll
                    for (int r = 0; r < RU; ++r) idx[r] = 1u;
#pragma unroll
                    for (int d = 0; d < D; ++d) {
#pragma unroll
                        for (int r = 0; r < RU; ++r) idx[r] = descend(idx[r], tw[idx[r]], xlo, xhi[r]);
                    }
#pragma unroll
                    for (int r = 0; r < RU; ++r) acc[r] = __fadd_rn(acc[r], __uint_as_float(tw[idx[r]]));
                }
            }
            if (!resident) {
                __syncthreads();   // every warp is done with stage s
                if (tid == 0 && g + stages < total_loads) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(g + stages);
                }
            }
        }

        if (active) {
            bool clamped = false;
            if (m <= ni) {
#pragma unroll
                for (int r = 0; r < RU; ++r) {
                    const int u = u0 + r;
                    if (u < p.F) {
                        const float v = acc[r];
                        float c = v;
                        if (isnan(v)) c = 0x1p-4f;
                        else c = fminf(fmaxf(v, 0x1p-4f), 0x1p17f);
                        clamped |= isnan(v) || c != v;
                        p.ips[((size_t)i * p.F + u) * p.H + (m - 1)] = c;
                    }
                }
            }
            if (__any_sync(0xffffffffu, clamped) && lane == 0) atomicOr(p.status + i, (uint32_t)TP_ST_IPS_CLAMPED);
        }
    }
}

template <int D, int RU>
int launch_d(const K2Params& p, cudaStream_t s) {
    const int TW = (2 << D) < 4 ? 4 : (2 << D);
    const int tree_bytes = TW * 4;
    int TC = std::max(1, std::min(std::max(p.n_trees, 1), kChunkBytes / tree_bytes));
    const int nchunks = p.n_trees == 0 ? 0 : (p.n_trees + TC - 1) / TC;
    const int stages = nchunks == 1 ? 1 : 2;
    const size_t smem = (size_t)stages * TC * tree_bytes;
    auto kern = k2_gbdt<D, RU>;
    int dev = 0, sms = 0, per_sm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return TP_ECUDA;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return TP_ECUDA;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return TP_ECUDA;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem) != cudaSuccess) return TP_ECUDA;
    const int grid = std::max(1, sms * std::max(1, per_sm));
    kern<<<grid, kThreads, smem, s>>>(p, TC, nchunks);
    return cudaPeekAtLastError() == cudaSuccess ? TP_OK : TP_ECUDA;
}

template <int RU>
int launch_ru(const K2Params& p, cudaStream_t s) {
    switch (p.depth) {
        case 0: return launch_d<0, RU>(p, s);
        case 1: return launch_d<1, RU>(p, s);
        case 2: return launch_d<2, RU>(p, s);
        case 3: return launch_d<3, RU>(p, s);
        case 4: return launch_d<4, RU>(p, s);
        case 5: return launch_d<5, RU>(p, s);
        case 6: return launch_d<6, RU>(p, s);
        case 7: return launch_d<7, RU>(p, s);
        case 8: return launch_d<8, RU>(p, s);
        case 9: return launch_d<9, RU>(p, s);
        case 10: return launch_d<10, RU>(p, s);
        case 11: return launch_d<11, RU>(p, s);
        case 12: return launch_d<12, RU>(p, s);
        default: return TP_EFORMAT;
    }
}

}  // namespace

int launch_gbdt(const K2Params& p, cudaStream_t s) {
    if (p.n_inst == 0) return TP_OK;
    if (p.F <= 2) return launch_ru<2>(p, s);
    if (p.F <= 4) return launch_ru<4>(p, s);
    return launch_ru<8>(p, s);
}

}  // namespace tp
