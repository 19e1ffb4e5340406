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
//  * One tree level costs 5 instructions per row: LDS (word), PRMT (pick the split feature's rank
//    into the upper half), IADD3 with carry-out (rank + 0xFFFF - j overflows <=> go right),
//    IADD3.X (idx = 2*idx + carry) and the IMAD that turns idx into the next word's shared-memory
//    address.  No branches, no divergence.
//  * Persistent-style grid (#SMs x occupancy CTAs); tiles are split evenly over CTAs by a
//    per-CTA scan of the per-instance tile counts.
#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include "tp_internal.cuh"

namespace tp {
namespace {

constexpr int kMaxThreads = 384;        // CTA size is a launch parameter (256 or 384 threads)
constexpr int kMaxWarps = kMaxThreads / 32;
// measured best (tools/k2_sweep.py, tools/k2_cells_sweep.py on C2 / C3)
constexpr int kDefaultThreads = 384, kDefaultThreadsRuns = 128, kDefaultThreadsCells = 256;
constexpr int kDefaultChunkBytes = 48 * 1024, kDefaultChunkBytesRuns = 16 * 1024, kDefaultChunkBytesCells = 32 * 1024;
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

__device__ __forceinline__ uint32_t prmt(uint32_t lo, uint32_t hi, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(lo), "r"(hi), "r"(sel));
    return r;
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

// Same step with the doubled index given: returns base2 + go_right (base2 = 2 * idx).
__device__ __forceinline__ uint32_t step_from(uint32_t base2, uint32_t w, uint32_t xlo, uint32_t xhi) {
    uint32_t out;
    asm("{\n\t.reg .b32 pr, t;\n\t"
        "prmt.b32 pr, %1, %2, %3;\n\t"
        "add.cc.u32 t, pr, %3;\n\t"
        "addc.u32 %0, %4, 0;\n\t}"
        : "=r"(out)
        : "r"(xlo), "r"(xhi), "r"(w), "r"(base2));
    return out;
}

// K3c's T' table entry of one (cell, level): int64 ticks of 2^-40 s, or, with the model's
// tick_shift = 8, uint32 units of 2^8 ticks (exact: see Model::tick_shift)
__device__ __forceinline__ void store_ticks(const K2Params& p, size_t at, float ips) {
    const long long t = ticks_of(ips);
    if (p.tick_shift) reinterpret_cast<uint32_t*>(p.lut_ticks)[at] = (uint32_t)(t >> p.tick_shift);
    else p.lut_ticks[at] = t;
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


enum Mode : int { kDirect = 0, kRuns = 1, kCells = 2 };
int env_int(const char* name, int dflt, int lo, int hi, int mult);

// Trees unrolled per step in cell mode (RU = 2 rows per lane -> 2 * UT independent descents).
#ifndef TP_K2_UT_CELLS
#define TP_K2_UT_CELLS 4
#endif
constexpr int kUnrollTreesCells = TP_K2_UT_CELLS;

// Work units.  Direct: one unit = one warp tile = 32 consecutive iterations x RU levels of one
// instance (ceil(n/32) * G units per instance).  Runs: one unit = one lane task = one run x RU
// levels (h * G per instance), packed 32 per warp tile across instance boundaries.  Cells: one unit
// = one distinct cell x RU levels (n_cells * G in total), no instance structure.
template <int MODE>
__device__ __forceinline__ int64_t units_of(const K2Params& p, int i, int G) {
    if (p.status[i] & p.skip) return 0;
    return MODE == kRuns ? (int64_t)p.run_h[i] * G : (int64_t)((p.n[i] + 31) >> 5) * G;
}

// ---------------------------------------------------------------------------------------------
// K2a (runs / cells): per instance, the runs of consecutive iterations m whose (batch, KV)
// features have the same ranks among the ensemble's thresholds -- M is constant on each run
// because tp and f are fixed per (instance, level).  One CTA per instance: keys for all m in
// shared memory (cut lists staged in shared memory when they fit), then a block-wide ballot
// compaction of the run heads.  Cell mode also claims each run's cell (rank_tp, rank_B,
// rank_KV) in a dense table and appends first-seen cells to the cell list.
constexpr int kRunsThreads = 256;

__global__ void __launch_bounds__(kRunsThreads)
k2_runs(const __grid_constant__ K2Params p) {
    extern __shared__ uint32_t skey[];               // [H + 1]: key of iteration m at skey[m]
    __shared__ int swarp[kRunsThreads / 32], swarp_ex[kRunsThreads / 32 + 1];
    const int i = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = (p.status[i] & p.skip) ? 0 : p.n[i];
    if (n == 0) {
        if (tid == 0) p.run_h[i] = 0;
        return;
    }
    const int nB = p.cut_off[2] - p.cut_off[1], nKV = p.cut_off[3] - p.cut_off[2];
    // rank tables (exact for integer features, L1-resident), a binary search beyond them
    const int lB = p.rtab_len[0], lKV = p.rtab_len[1];
    const uint16_t* tB = p.rtab + p.rtab_off[0];
    const uint16_t* tKV = p.rtab + p.rtab_off[1];
    const bool cells = p.cell_tab != nullptr;
    uint32_t cell_base = 0;
    if (cells) {
        const uint32_t rtp = rank_of(p.cuts + p.cut_off[0], p.cut_off[1] - p.cut_off[0], (float)p.inst[i].tp);
        cell_base = rtp * (uint32_t)(nB + 1) * (uint32_t)(nKV + 1);
    }
    const size_t row = (size_t)i * p.H;
    for (int m = 1 + tid; m <= n; m += kRunsThreads) {
        const int b = p.B[row + m - 1], kv = p.KV[row + m - 1];
        const uint32_t rb = b < lB ? __ldg(tB + b) : rank_of(p.cuts + p.cut_off[1], nB, (float)b);
        const uint32_t rk = kv < lKV ? __ldg(tKV + kv) : rank_of(p.cuts + p.cut_off[2], nKV, (float)kv);
        skey[m] = cells ? cell_base + rb * (uint32_t)(nKV + 1) + rk : (rb | (rk << 16));
    }
    __syncthreads();
    int base = 0;
    for (int m0 = 1; m0 <= n; m0 += kRunsThreads) {
        const int m = m0 + tid;
        const bool head = m <= n && (m == 1 || skey[m] != skey[m - 1]);
        const unsigned mask = __ballot_sync(0xffffffffu, head);
        if (lane == 0) swarp[warp] = __popc(mask);
        __syncthreads();
        if (tid < 32) {      // exclusive scan of the 8 warp counts (one warp)
            const int c = lane < kRunsThreads / 32 ? swarp[lane] : 0;
            int x = c;
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane < kRunsThreads / 32) swarp_ex[lane] = x - c;
            if (lane == kRunsThreads / 32 - 1) swarp_ex[kRunsThreads / 32] = x;
        }
        __syncthreads();
        const int before = base + swarp_ex[warp];
        if (head) {
            const int pos = before + __popc(mask & ((1u << lane) - 1u));
            const uint32_t key = skey[m];
            p.run_m[row + pos] = m;
            p.run_key[row + pos] = key;
            // first claimant of a cell appends it to the list; the LUT row index is published in
            // cell_tab after the claim and read only by later kernels
            if (cells && __ldcg(p.cell_tab + key) == -1 && atomicCAS(p.cell_tab + key, -1, -2) == -1) {
                const int idx = atomicAdd(p.cell_count, 1) + 1;   // cell_count holds count - 1
                p.cell_list[idx] = key;
                p.cell_clamp[key] = 0u;
                p.cell_tab[key] = idx;
            }
        }
        base += swarp_ex[kRunsThreads / 32];
        __syncthreads();
    }
    if (tid == 0) p.run_h[i] = base;
}

// ---------------------------------------------------------------------------------------------
// K2c (cells): every iteration of every run gets its cell's LUT row; IPS_CLAMPED from the
// per-cell clamp masks.  One CTA per instance; run starts in shared memory; the stores of one
// level are coalesced over consecutive iterations.
constexpr int kExpandThreads = 256;

__global__ void __launch_bounds__(kExpandThreads)
k2_expand(const __grid_constant__ K2Params p) {
    extern __shared__ int sx[];     // [h] run starts, [h] LUT rows
    const int i = blockIdx.x, tid = threadIdx.x;
    const int h = p.run_h[i];
    if (h == 0) return;
    const int n = p.n[i];
    const size_t row = (size_t)i * p.H;
    int* sm = sx;
    int* sidx = sx + h;
    bool clamped = false;
    for (int k = tid; k < h; k += kExpandThreads) {
        sm[k] = p.run_m[row + k];
        const uint32_t key = p.run_key[row + k];
        sidx[k] = p.cell_tab[key];
        clamped |= p.cell_clamp[key] != 0;
    }
    if (__syncthreads_or(clamped) && tid == 0) atomicOr(p.status + i, (uint32_t)TP_ST_IPS_CLAMPED);
    const int F = p.F;
    for (int m = 1 + tid; m <= n; m += kExpandThreads) {
        int lo = 0, hi = h;     // last run with start <= m
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (sm[mid] <= m) lo = mid;
            else hi = mid;
        }
        const float* lrow = p.lut + (size_t)sidx[lo] * F;
        for (int u = 0; u < F; ++u) p.ips[(row * F) + (size_t)u * p.H + (m - 1)] = __ldg(lrow + u);
    }
}

// ---------------------------------------------------------------------------------------------
// K2b: tree-ensemble evaluation (all modes)
template <int D, int RU, int MODE>
__global__ void __launch_bounds__(kMaxThreads, 2)
k2_gbdt(const __grid_constant__ K2Params p, int TC, int nchunks) {
    extern __shared__ __align__(128) uint32_t sw[];
    __shared__ __align__(8) uint64_t full[2];
    __shared__ int64_t red[kMaxWarps];
    __shared__ int64_t s_start_pc;
    __shared__ int s_start_i;
    __shared__ uint32_t s_rf[kMaxF];

    constexpr int TW = (2 << D) < 4 ? 4 : (2 << D);    // words per tree (>= 16 B for TMA)
    constexpr int UPT = MODE == kDirect ? 1 : 32;      // units per warp tile
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nthreads = blockDim.x, nwarps = nthreads >> 5;
    const int G = (p.F + RU - 1) / RU;
    const int I = p.n_inst;
    const bool resident = nchunks == 1;
    const int stages = resident ? 1 : 2;
    const int chunk_words = TC * TW;
    const float* cutsB = p.cuts + p.cut_off[1];
    const float* cutsKV = p.cuts + p.cut_off[2];
    const float* cutsTP = p.cuts + p.cut_off[0];
    const int nB = p.cut_off[2] - p.cut_off[1], nKV = p.cut_off[3] - p.cut_off[2], nTP = p.cut_off[1] - p.cut_off[0];

    if (tid < p.F)
        s_rf[tid] = rank_of(p.cuts + p.cut_off[3], p.cut_off[4] - p.cut_off[3], p.freq[tid]);

    // ---- split the tile space [0, ceil(U / UPT)) evenly over CTAs ----
    int64_t U = 0;
    int ncell = 0;
    if constexpr (MODE == kCells) {
        ncell = *p.cell_count + 1;
        U = (int64_t)ncell * G;
    } else {
        for (int i = tid; i < I; i += nthreads) U += units_of<MODE>(p, i, G);
        for (int o = 16; o; o >>= 1) U += __shfl_xor_sync(0xffffffffu, U, o);
        if (lane == 0) red[warp] = U;
        __syncthreads();
        U = 0;
        for (int k = 0; k < nwarps; ++k) U += red[k];
    }
    const int64_t ntiles = (U + UPT - 1) / UPT;
    const int64_t t0 = ntiles * blockIdx.x / gridDim.x, t1 = ntiles * (blockIdx.x + 1) / gridDim.x;
    if (t0 >= t1) return;   // uniform: no work for this CTA
    const int64_t u_first = t0 * UPT;

    // locate the instance holding unit u_first (block-wide scan over instances, chunk by chunk)
    if (tid == 0) {
        s_start_i = MODE == kCells ? 0 : -1;
        s_start_pc = 0;
    }
    __syncthreads();
    if constexpr (MODE != kCells) {
        int64_t base_pc = 0;
        for (int c0 = 0; c0 < I; c0 += nthreads) {
            const int i = c0 + tid;
            const int64_t v = i < I ? units_of<MODE>(p, i, G) : 0;
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
            if (i < I && v > 0 && excl <= u_first && u_first < incl) {
                s_start_i = i;
                s_start_pc = excl;
            }
            for (int k = 0; k < nwarps; ++k) base_pc += red[k];
            __syncthreads();
            if (s_start_i >= 0) break;
        }
    }

    if (tid == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int nrounds = (int)((t1 - t0 + nwarps - 1) / nwarps);
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
    int64_t pc = s_start_pc;   // units before instance ci
    int64_t g = 0;             // loads consumed so far

    for (int round = 0; round < nrounds; ++round) {
        const int64_t t = t0 + (int64_t)round * nwarps + warp;
        const bool active = t < t1;
        int i = 0, m = 0, u0 = 0, ni = 0, m_end = 0, cidx = -1;
        uint32_t cell_id = 0;
        uint32_t xlo = 0, xhi[RU];
        float acc[RU];
        if (active) {
            const int64_t ub = t * UPT;   // first unit of the tile
            uint32_t rkv = 0;
            if constexpr (MODE == kCells) {
                // lane task = unit ub + lane -> (cell row idx, level group ug)
                const int64_t uu = ub + lane;
                if (uu < U) {
                    const int ug = (int)(uu / ncell);
                    cidx = (int)(uu - (int64_t)ug * ncell);
                    u0 = ug * RU;
                    const uint32_t c = p.cell_list[cidx];
                    cell_id = c;
                    const uint32_t nk1 = (uint32_t)nKV + 1, nb1 = (uint32_t)nB + 1;
                    rkv = c % nk1;
                    const uint32_t rb = (c / nk1) % nb1, rtp = c / (nk1 * nb1);
                    xlo = rtp | (rb << 16);
                }
            } else {
                int64_t ti;
                while (ub >= pc + (ti = units_of<MODE>(p, ci, G)) && ci < I - 1) {
                    pc += ti;
                    ++ci;
                }
                if constexpr (MODE == kRuns) {
                    // lane task = unit ub + lane -> (instance li, run k, level group ug); the tile's
                    // lanes may span several instances (each lane walks on from the warp's cursor)
                    const int64_t uu = ub + lane;
                    int li = ci;
                    int64_t lpc = pc, lt;
                    while (uu >= lpc + (lt = units_of<MODE>(p, li, G)) && li < I - 1) {
                        lpc += lt;
                        ++li;
                    }
                    i = li;
                    uint32_t key = 0;
                    m = 0x7fffffff;
                    if (uu < U) {
                        const int h = p.run_h[i];
                        const int tau = (int)(uu - lpc);
                        const int ug = tau / h, k = tau - ug * h;
                        u0 = ug * RU;
                        key = p.run_key[(size_t)i * p.H + k];
                        m = p.run_m[(size_t)i * p.H + k];
                        ni = p.n[i];
                        m_end = (k + 1 < h) ? p.run_m[(size_t)i * p.H + k + 1] : ni + 1;
                    }
                    xlo = rank_of(cutsTP, nTP, (float)p.inst[i].tp) | ((key & 0xFFFFu) << 16);
                    rkv = key >> 16;
                } else {
                    i = ci;
                    const int64_t tau = ub - pc;
                    const int mt = (int)(tau / G), ug = (int)(tau % G);
                    ni = p.n[i];
                    u0 = ug * RU;
                    m = mt * 32 + lane + 1;
                    int bv = 0, kvv = 0;
                    if (m <= ni) {
                        bv = p.B[(size_t)i * p.H + m - 1];
                        kvv = p.KV[(size_t)i * p.H + m - 1];
                    }
                    const uint32_t rb = bv < p.rtab_len[0] ? p.rtab[p.rtab_off[0] + bv] : rank_of(cutsB, nB, (float)bv);
                    rkv = kvv < p.rtab_len[1] ? p.rtab[p.rtab_off[1] + kvv] : rank_of(cutsKV, nKV, (float)kvv);
                    xlo = rank_of(cutsTP, nTP, (float)p.inst[i].tp) | (rb << 16);
                }
            }
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
                // one tree for the lane's RU rows; descents of different trees are independent
                // (only the fp32 accumulation is ordered), so unrolling over trees adds ILP
                auto tree = [&](int tt) {
                    const uint32_t* tw = cw + tt * TW;
                    uint32_t idx[RU];
                    if constexpr (D >= 2) {
                        // levels 0-1: the root and both of its children are shared by all RU rows
                        // of the lane (one LDS.128 of words 0..3); the level-0 carry selects the
                        // level-1 word directly.
                        const uint32_t w1 = tw[1];
                        const uint2 w23 = *reinterpret_cast<const uint2*>(tw + 2);
#pragma unroll
                        for (int r = 0; r < RU; ++r) {
                            const bool c0 = prmt(xlo, xhi[r], w1) > ~w1;    // carry-out of prmt + w1
                            idx[r] = step_from(c0 ? 6u : 4u, c0 ? w23.y : w23.x, xlo, xhi[r]);
                        }
                    } else {
#pragma unroll
                        for (int r = 0; r < RU; ++r) idx[r] = 1u;
                    }
#pragma unroll
                    for (int d = (D >= 2 ? 2 : 0); d < D; ++d) {
#pragma unroll
                        for (int r = 0; r < RU; ++r) idx[r] = descend(idx[r], tw[idx[r]], xlo, xhi[r]);
                    }
#pragma unroll
                    for (int r = 0; r < RU; ++r) acc[r] = __fadd_rn(acc[r], __uint_as_float(tw[idx[r]]));
                };
                if constexpr (MODE == kCells) {
#pragma unroll kUnrollTreesCells
                    for (int tt = 0; tt < nt; ++tt) tree(tt);
                } else {
                    for (int tt = 0; tt < nt; ++tt) tree(tt);
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
            uint32_t cmask = 0;
#pragma unroll
            for (int r = 0; r < RU; ++r) {
                const float v = acc[r];
                const float c = isnan(v) ? 0x1p-4f : fminf(fmaxf(v, 0x1p-4f), 0x1p17f);
                if (u0 + r < p.F && (isnan(v) || c != v)) cmask |= 1u << (u0 + r);
                acc[r] = c;
            }
            if constexpr (MODE == kCells) {
                if (cidx >= 0) {
#pragma unroll
                    for (int r = 0; r < RU; ++r)
                        if (u0 + r < p.F) {
                            p.lut[(size_t)cidx * p.F + u0 + r] = acc[r];
                            store_ticks(p, (size_t)cell_id * p.F + u0 + r, acc[r]);
                        }
                    if (cmask) atomicOr(p.cell_clamp + cell_id, cmask);
                }
            } else if constexpr (MODE == kRuns) {
                // the lane writes its run [m, m_end) for its RU levels
                for (int mm = m; mm < m_end; ++mm) {
#pragma unroll
                    for (int r = 0; r < RU; ++r)
                        if (u0 + r < p.F) p.ips[((size_t)i * p.F + u0 + r) * p.H + (mm - 1)] = acc[r];
                }
                if (cmask && m <= ni) atomicOr(p.status + i, (uint32_t)TP_ST_IPS_CLAMPED);
            } else {
                if (m <= ni) {
#pragma unroll
                    for (int r = 0; r < RU; ++r)
                        if (u0 + r < p.F) p.ips[((size_t)i * p.F + u0 + r) * p.H + (m - 1)] = acc[r];
                }
                if (__any_sync(0xffffffffu, cmask != 0 && m <= ni) && lane == 0)
                    atomicOr(p.status + i, (uint32_t)TP_ST_IPS_CLAMPED);
            }
        }
    }
}

// ---------------------------------------------------------------------------------------------
// K2p (cell mode, tree-resident phases): the ensemble is cut into phases of consecutive trees that
// fit in one SM's shared memory (<= ~200 KB); one launch per phase, one CTA per SM.  Each CTA
// TMA-loads its phase once (one mbarrier per 8-tree chunk, so descents start as soon as the first
// chunk lands; no buffer is ever reused, so no __syncthreads after the prologue) and evaluates its
// contiguous share of the (cell, level-group) tasks for every tree of the phase.  The running fp32
// sum of a row is carried from phase to phase in the LUT itself (the first phase starts from the
// base score, the last one clamps, writes the tick LUT and the clamp masks), so every row's leaves
// are still added one by one in tree order (reading A-7).
constexpr int kPhaseChunkTrees = 8;
#ifndef TP_K2_TPAIR
#define TP_K2_TPAIR 1
#endif
constexpr int kMaxPhaseChunks = 64;
constexpr int kPhaseThreads = 1024;

template <int D, int RU>
__global__ void __launch_bounds__(kPhaseThreads, 1)
k2_cells_phase(const __grid_constant__ K2Params p, int t_begin, int t_count, int first, int last) {
    extern __shared__ __align__(128) uint32_t sw[];
    __shared__ __align__(8) uint64_t bar[kMaxPhaseChunks];
    __shared__ uint32_t s_rf[kMaxF];
    constexpr int TW = (2 << D) < 4 ? 4 : (2 << D);
    const int tid = threadIdx.x;
    const int G = (p.F + RU - 1) / RU;
    const int nchunks = (t_count + kPhaseChunkTrees - 1) / kPhaseChunkTrees;
    // the phase's trees are model constants: their TMA loads are issued before waiting on the
    // previous kernel (programmatic dependent launch), overlapping its tail
    if (tid == 0) {
        for (int c = 0; c < nchunks; ++c) mbar_init(&bar[c], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int c = 0; c < nchunks; ++c) {
            const int nt = min(kPhaseChunkTrees, t_count - c * kPhaseChunkTrees);
            const uint32_t bytes = (uint32_t)nt * TW * 4u;
            mbar_expect_tx(&bar[c], bytes);
            tma_load(sw + (size_t)c * kPhaseChunkTrees * TW, p.words + (size_t)(t_begin + c * kPhaseChunkTrees) * TW,
                     bytes, &bar[c]);
        }
    }
    if (tid < p.F) s_rf[tid] = rank_of(p.cuts + p.cut_off[3], p.cut_off[4] - p.cut_off[3], p.freq[tid]);
    __syncthreads();                           // barriers initialised, s_rf visible
    pdl_wait();                                // cell list / LUT of the previous kernel
    const int ncell = *p.cell_count + 1;
    const int64_t U = (int64_t)ncell * G;
    const int64_t t0 = U * blockIdx.x / gridDim.x, t1 = U * (blockIdx.x + 1) / gridDim.x;
    const int nB = p.cut_off[2] - p.cut_off[1], nKV = p.cut_off[3] - p.cut_off[2];
    const uint32_t nk1 = (uint32_t)nKV + 1, nb1 = (uint32_t)nB + 1;
    // One work item = RR rows of one cell (levels u0 .. u0 + RR - 1), all trees of the phase.
    auto item = [&](auto rr_tag, int cidx, int u0) {
        constexpr int RR = decltype(rr_tag)::value;
        const uint32_t c = p.cell_list[cidx];
        const uint32_t rkv = c % nk1;
        const uint32_t rb = (c / nk1) % nb1, rtp = c / (nk1 * nb1);
        const uint32_t xlo = rtp | (rb << 16);
        uint32_t xhi[RR];
        float acc[RR];
#pragma unroll
        for (int r = 0; r < RR; ++r) {
            const int u = min(u0 + r, p.F - 1);
            xhi[r] = rkv | (s_rf[u] << 16);
            acc[r] = first ? p.base : p.lut[(size_t)cidx * p.F + u];
        }
        for (int ch = 0; ch < nchunks; ++ch) {
            mbar_wait(&bar[ch], 0u);
            const uint32_t* cw = sw + (size_t)ch * kPhaseChunkTrees * TW;
            const int nt = min(kPhaseChunkTrees, t_count - ch * kPhaseChunkTrees);
            auto tree = [&](int tt) {
                const uint32_t* tw = cw + tt * TW;
                uint32_t idx[RR];
                if constexpr (D >= 2) {
                    const uint32_t w1 = tw[1];
                    const uint2 w23 = *reinterpret_cast<const uint2*>(tw + 2);
#pragma unroll
                    for (int r = 0; r < RR; ++r) {
                        const bool c0 = prmt(xlo, xhi[r], w1) > ~w1;
                        idx[r] = step_from(c0 ? 6u : 4u, c0 ? w23.y : w23.x, xlo, xhi[r]);
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < RR; ++r) idx[r] = 1u;
                }
#pragma unroll
                for (int d = (D >= 2 ? 2 : 0); d < D; ++d) {
#pragma unroll
                    for (int r = 0; r < RR; ++r) idx[r] = descend(idx[r], tw[idx[r]], xlo, xhi[r]);
                }
#pragma unroll
                for (int r = 0; r < RR; ++r) acc[r] = __fadd_rn(acc[r], __uint_as_float(tw[idx[r]]));
            };
            // TP_K2_TPAIR: two trees' descents interleaved level by level (2 x RR independent
            // dependent-load chains per thread), then their leaves added in tree order -- the same
            // fp32 sum, more latency hidden when there are few rows per SM
            auto tree2 = [&](int tt) {
                const uint32_t* ta = cw + tt * TW;
                const uint32_t* tb = ta + TW;
                uint32_t ia[RR], ib[RR];
                if constexpr (D >= 2) {
                    const uint32_t a1 = ta[1], b1 = tb[1];
                    const uint2 a23 = *reinterpret_cast<const uint2*>(ta + 2);
                    const uint2 b23 = *reinterpret_cast<const uint2*>(tb + 2);
#pragma unroll
                    for (int r = 0; r < RR; ++r) {
                        const bool ca = prmt(xlo, xhi[r], a1) > ~a1;
                        const bool cb = prmt(xlo, xhi[r], b1) > ~b1;
                        ia[r] = step_from(ca ? 6u : 4u, ca ? a23.y : a23.x, xlo, xhi[r]);
                        ib[r] = step_from(cb ? 6u : 4u, cb ? b23.y : b23.x, xlo, xhi[r]);
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < RR; ++r) ia[r] = ib[r] = 1u;
                }
#pragma unroll
                for (int d = (D >= 2 ? 2 : 0); d < D; ++d) {
#pragma unroll
                    for (int r = 0; r < RR; ++r) {
                        ia[r] = descend(ia[r], ta[ia[r]], xlo, xhi[r]);
                        ib[r] = descend(ib[r], tb[ib[r]], xlo, xhi[r]);
                    }
                }
#pragma unroll
                for (int r = 0; r < RR; ++r) {
                    acc[r] = __fadd_rn(acc[r], __uint_as_float(ta[ia[r]]));
                    acc[r] = __fadd_rn(acc[r], __uint_as_float(tb[ib[r]]));
                }
            };
            if (nt == kPhaseChunkTrees) {
                if constexpr (TP_K2_TPAIR) {
#pragma unroll
                    for (int tt = 0; tt < kPhaseChunkTrees; tt += 2) tree2(tt);
                } else {
#pragma unroll
                    for (int tt = 0; tt < kPhaseChunkTrees; ++tt) tree(tt);
                }
            } else {
                for (int tt = 0; tt < nt; ++tt) tree(tt);
            }
        }
        if (last) {
            uint32_t cmask = 0;
#pragma unroll
            for (int r = 0; r < RR; ++r) {
                const float v = acc[r];
                const float cl = isnan(v) ? 0x1p-4f : fminf(fmaxf(v, 0x1p-4f), 0x1p17f);
                if (u0 + r < p.F) {
                    if (isnan(v) || cl != v) cmask |= 1u << (u0 + r);
                    p.lut[(size_t)cidx * p.F + u0 + r] = cl;
                    if (p.lut_ticks) store_ticks(p, (size_t)c * p.F + u0 + r, cl);
                }
            }
            if (cmask) atomicOr(p.cell_clamp + c, cmask);
        } else {
#pragma unroll
            for (int r = 0; r < RR; ++r)
                if (u0 + r < p.F) p.lut[(size_t)cidx * p.F + u0 + r] = acc[r];
        }
    };
    // The CTA's RU-row tasks [t0, t1): the first P (a multiple of 4 SMSPs x 32 lanes) run as
    // RU-row items, so every SMSP gets the same number of warp-items; with RU = 2 the remaining
    // tasks run as single-row items (two per task), so the ragged end costs half-size warp-items
    // instead of one more full round on some SMSPs.
    const int64_t ntask = t1 - t0;
    const int64_t P = (RU == 2) ? (ntask / 128) * 128 : ntask;
    const int64_t nitems = P + (ntask - P) * (RU == 2 ? 2 : 0);
    for (int64_t it = tid; it < nitems; it += blockDim.x) {   // (no item: the CTA still drains its TMA)
        if (it < P) {                                         // warp-uniform: P is a multiple of 32
            const int64_t task = t0 + it;
            const int ug = (int)(task / ncell);
            const int cidx = (int)(task - (int64_t)ug * ncell);
            item(std::integral_constant<int, RU>{}, cidx, ug * RU);
        } else if constexpr (RU == 2) {
            const int64_t s1 = it - P;
            const int64_t task = t0 + P + (s1 >> 1);
            const int ug = (int)(task / ncell);
            const int cidx = (int)(task - (int64_t)ug * ncell);
            item(std::integral_constant<int, 1>{}, cidx, ug * 2 + (int)(s1 & 1));
        }
    }
    if (tid == 0 && nitems == 0)               // no task: wait for the bulk copies before exiting
        for (int ch = 0; ch < nchunks; ++ch) mbar_wait(&bar[ch], 0u);
}

template <int D, int RU>
int launch_phases(const K2Params& p, cudaStream_t s) {
    const int TW = (2 << D) < 4 ? 4 : (2 << D);
    const int tree_bytes = TW * 4;
    static const int budget = env_int("TP_K2_PHASE_KB", 200, 8, 220, 1) * 1024;
    const int max_trees = std::max(1, std::min(budget / tree_bytes, kMaxPhaseChunks * kPhaseChunkTrees));
    const int nphase = p.n_trees == 0 ? 1 : (p.n_trees + max_trees - 1) / max_trees;
    const int per = p.n_trees == 0 ? 0 : (p.n_trees + nphase - 1) / nphase;   // balanced phases
    const size_t smem = (size_t)std::max(per, 1) * tree_bytes;
    auto kern = k2_cells_phase<D, RU>;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return TP_ECUDA;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return TP_ECUDA;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return TP_ECUDA;
    for (int ph = 0; ph < nphase; ++ph) {
        const int tb = ph * per, tc = std::max(0, std::min(per, p.n_trees - tb));
        if (launch_pdl(kern, dim3(sms), dim3(kPhaseThreads), smem, s, p, tb, tc, (int)(ph == 0),
                       (int)(ph == nphase - 1)) != cudaSuccess)
            return TP_ECUDA;
    }
    return TP_OK;
}

// Tuning knobs (read once): TP_K2_THREADS (CTA size, multiple of 32), TP_K2_CHUNK_KB (tree chunk).
int env_int(const char* name, int dflt, int lo, int hi, int mult) {
    const char* v = std::getenv(name);
    if (!v) return dflt;
    const int x = std::atoi(v);
    return (x >= lo && x <= hi && x % mult == 0) ? x : dflt;
}

bool set_smem_attr(const void* fn, int bytes, bool* done, int dev) {
    if (dev < 64 && done[dev]) return true;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
    if (dev < 64) done[dev] = true;
    return true;
}

template <int D, int RU, int MODE>
int launch_d(const K2Params& p, cudaStream_t s) {
    const int TW = (2 << D) < 4 ? 4 : (2 << D);
    const int tree_bytes = TW * 4;
    static const int threads =
        env_int("TP_K2_THREADS",
                MODE == kDirect ? kDefaultThreads : MODE == kRuns ? kDefaultThreadsRuns : kDefaultThreadsCells, 64,
                kMaxThreads, 32);
    static const int chunk_bytes =
        env_int("TP_K2_CHUNK_KB",
                (MODE == kDirect ? kDefaultChunkBytes : MODE == kRuns ? kDefaultChunkBytesRuns : kDefaultChunkBytesCells) /
                    1024,
                4, 100, 1) *
        1024;
    int TC = std::max(1, std::min(std::max(p.n_trees, 1), chunk_bytes / tree_bytes));
    const int nchunks = p.n_trees == 0 ? 0 : (p.n_trees + TC - 1) / TC;
    const int stages = nchunks == 1 ? 1 : 2;
    const size_t smem = (size_t)stages * TC * tree_bytes;
    auto kern = k2_gbdt<D, RU, MODE>;
    int dev = 0, sms = 0, per_sm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return TP_ECUDA;
    if (MODE != kDirect && !p.runs_ready) {
        static bool runs_attr[64] = {};
        if (!set_smem_attr((const void*)k2_runs, (kMaxH + 1) * 4, runs_attr, dev)) return TP_ECUDA;
        if (MODE == kCells) {
            if (cudaMemsetAsync(p.cell_count, 0xFF, 4 + (size_t)p.n_cells * 4, s) != cudaSuccess)   // + cell_tab
                return TP_ECUDA;
        }
        k2_runs<<<p.n_inst, kRunsThreads, (size_t)(p.H + 1) * 4, s>>>(p);
        if (cudaPeekAtLastError() != cudaSuccess) return TP_ECUDA;
    }
    static const bool chunked = env_int("TP_K2_CELLS_CHUNKED", 0, 0, 1, 1) == 1;
    if (MODE == kCells && !chunked && RU <= 2) {
        // tree-resident phases (the chunked kernel below stays selectable for comparisons)
        const int rc = launch_phases<D, RU>(p, s);
        if (rc != TP_OK) return rc;
    } else {
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return TP_ECUDA;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return TP_ECUDA;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess) return TP_ECUDA;
    const int grid = std::max(1, sms * std::max(1, per_sm));
    kern<<<grid, threads, smem, s>>>(p, TC, nchunks);
    if (cudaPeekAtLastError() != cudaSuccess) return TP_ECUDA;
    }
    if (MODE == kCells && p.ips) {   // ips == NULL: values stay in the LUT (tp_select_freq_ws)
        static bool exp_attr[64] = {};
        if (!set_smem_attr((const void*)k2_expand, 2 * kMaxH * 4, exp_attr, dev)) return TP_ECUDA;
        k2_expand<<<p.n_inst, kExpandThreads, (size_t)2 * p.H * 4, s>>>(p);
        if (cudaPeekAtLastError() != cudaSuccess) return TP_ECUDA;
    }
    return TP_OK;
}

template <int RU, int MODE>
int launch_ru(const K2Params& p, cudaStream_t s) {
    switch (p.depth) {
        case 0: return launch_d<0, RU, MODE>(p, s);
        case 1: return launch_d<1, RU, MODE>(p, s);
        case 2: return launch_d<2, RU, MODE>(p, s);
        case 3: return launch_d<3, RU, MODE>(p, s);
        case 4: return launch_d<4, RU, MODE>(p, s);
        case 5: return launch_d<5, RU, MODE>(p, s);
        case 6: return launch_d<6, RU, MODE>(p, s);
        case 7: return launch_d<7, RU, MODE>(p, s);
        case 8: return launch_d<8, RU, MODE>(p, s);
        case 9: return launch_d<9, RU, MODE>(p, s);
        case 10: return launch_d<10, RU, MODE>(p, s);
        case 11: return launch_d<11, RU, MODE>(p, s);
        case 12: return launch_d<12, RU, MODE>(p, s);
        default: return TP_EFORMAT;
    }
}

// Rows per lane: RU = 8 levels (fewer when F is small).  TP_K2_RU (2/4/8) overrides it per mode:
// fewer rows per lane = more warps for the same work (latency-bound small problems).
template <int MODE>
int launch_mode(const K2Params& p, cudaStream_t s) {
    static const int ru_env = env_int(MODE == kCells ? "TP_K2_RU_CELLS" : "TP_K2_RU", MODE == kCells ? 2 : 8, 1, 8, 1);
    const int ru = std::min(ru_env, p.F <= 2 ? 2 : p.F <= 4 ? 4 : 8);
    if constexpr (MODE == kCells) {
        if (ru == 1) return launch_ru<1, MODE>(p, s);
    }
    if (ru <= 2) return launch_ru<2, MODE>(p, s);
    if (ru <= 4) return launch_ru<4, MODE>(p, s);
    return launch_ru<8, MODE>(p, s);
}

uintptr_t align256(uintptr_t x) { return (x + 255) & ~(uintptr_t)255; }

}  // namespace

int launch_gbdt(const K2Params& p, bool runs, cudaStream_t s) {
    if (p.n_inst == 0) return TP_OK;
    if (!runs) return launch_mode<kDirect>(p, s);
    return p.cell_tab ? launch_mode<kCells>(p, s) : launch_mode<kRuns>(p, s);
}

int64_t model_cells(const Model& m) {
    return (int64_t)(m.n_cuts[0] + 1) * (m.n_cuts[1] + 1) * (m.n_cuts[2] + 1);
}

// Workspace: run_h [I], run_m [I][H], run_key [I][H], end_n [I], end_d [I][H]
// (compact path); cell mode adds cell_tab [n_cells], cell_list [cap], cell_count, cell_clamp [n_cells],
// lut [cap][F] with cap = min(n_cells, I * H).  Returns the bytes used past `ws`.
static size_t carve(void* ws, int64_t n_cells, int32_t n_inst, int32_t H, int32_t F, K2Params& p) {
    const size_t I = (size_t)(n_inst > 0 ? n_inst : 1);
    const uintptr_t a0 = (uintptr_t)ws;
    uintptr_t a = align256(a0);
    p.run_h = reinterpret_cast<int32_t*>(a);
    a = align256(a + I * 4);
    p.run_m = reinterpret_cast<int32_t*>(a);
    a = align256(a + I * (size_t)H * 4);
    p.run_key = reinterpret_cast<uint32_t*>(a);
    a = align256(a + I * (size_t)H * 4);
    p.end_n = reinterpret_cast<int32_t*>(a);
    a = align256(a + I * 4);
    p.end_d = reinterpret_cast<long long*>(a);
    a = align256(a + I * (size_t)H * 8);
    p.flag_list = reinterpret_cast<int32_t*>(a);
    a = align256(a + I * 4);
    p.flag_count = nullptr;
    p.k3_next = nullptr;
    p.k1_next = nullptr;
    p.k3_done = nullptr;
    p.cell_tab = nullptr;
    p.cell_list = nullptr;
    p.cell_count = nullptr;
    p.cell_clamp = nullptr;
    p.lut = nullptr;
    p.lut_ticks = nullptr;
    p.n_cells = 0;
    p.cell_cap = 0;
    if (n_cells > 0 && n_cells <= kMaxCells) {
        const int64_t cap = std::min<int64_t>(n_cells, (int64_t)I * H);
        p.n_cells = (int32_t)n_cells;
        p.cell_cap = (int32_t)cap;
        // K3c's counters, flag_count and cell_count (all stored as count - 1) directly before
        // cell_tab: one 0xFF memset (K1c's launch) resets them all
        p.k1_next = reinterpret_cast<int32_t*>(a);
        p.k3_next = reinterpret_cast<int32_t*>(a + 4);
        p.k3_done = reinterpret_cast<int32_t*>(a + 8);
        p.flag_count = reinterpret_cast<int32_t*>(a + 12);
        p.cell_count = reinterpret_cast<int32_t*>(a + 16);
        p.cell_tab = reinterpret_cast<int32_t*>(a + 20);
        a = align256(a + 20 + (size_t)n_cells * 4);
        p.cell_list = reinterpret_cast<uint32_t*>(a);
        a = align256(a + (size_t)cap * 4);
        p.cell_clamp = reinterpret_cast<uint32_t*>(a);       // by cell id
        a = align256(a + (size_t)n_cells * 4);
        p.lut = reinterpret_cast<float*>(a);
        a = align256(a + (size_t)cap * F * 4);
        p.lut_ticks = reinterpret_cast<long long*>(a);       // by cell id: K3c indexes it by the piece's key
        a = align256(a + (size_t)n_cells * F * 8);
    }
    return (size_t)(a - a0);
}

size_t runs_workspace_bytes(int64_t n_cells, int32_t n_inst, int32_t H, int32_t F) {
    K2Params p{};
    return carve(nullptr, n_cells, n_inst, H, F, p) + 256;
}

void runs_workspace_carve(void* ws, int64_t n_cells, int32_t n_inst, int32_t H, int32_t F, K2Params& p) {
    carve(ws, n_cells, n_inst, H, F, p);
}

}  // namespace tp
