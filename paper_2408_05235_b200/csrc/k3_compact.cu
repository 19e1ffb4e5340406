// K3c -- the compact path's SLO scan and frequency choice: T' = 1/IPS (reading A-9),
// T_R = cumulative sum (Eq. 3, exact int64 ticks, reading A-10), TBT check, E2E
// check Eq. 4 and the lowest SLO-meeting frequency.
//
// One WARP per instance (or W warps at small batches), lane u = frequency level u (F <= 32).  K1c
// cut m = 1..n into PIECES (k1_compact.cu, piece_rules): runs of one cell -- so one T' per level --
// that also end at every request's last iteration, each with Dmin of its tail.  Every lane walks the
// same pieces in m order (warp-uniform control flow, only the T' value differs per lane):
//   T_R(tail) = T_R(previous tail) + len * T'[cell][u]        (exact: integers)
//   pass_u   &= T_R(tail) < Dmin(tail)                        (strict, Eq. 4; no deadline = INT64_MAX)
// so a piece is one fixed step: one broadcast shared-memory load of its staged record {LUT row, len,
// Dmin}, one load of the lane's T' from K2's tick LUT, a 64-bit multiply-add and a 64-bit compare.
// Records are loaded lane-parallel 32 pieces at a time (run_m / run_key / end_d, coalesced), staged
// in shared memory (double-buffered: the next chunk's loads are in flight while this one is walked)
// and walked in a fully unrolled 32-step loop that keeps the LUT loads of the next PD pieces in
// flight (the LUT is indexed by cell id, so a record needs no table lookup).  TBT: T_R[n] <= n * tbt_slo (tie passes).  The decision is one __ballot_sync
// over the levels' pass bits: __ffs of it (exhaustive, reading A-13) or the paper's binary search
// replayed on the bit vector (reading A-24).  IPS_CLAMPED: the OR of the pieces' cell clamp masks,
// restricted to the visited levels (all F in the exhaustive order).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "tp_internal.cuh"

namespace tp {
namespace {

constexpr int kWarpsPerCta = 8;
constexpr unsigned kFull = 0xffffffffu;
#ifndef TP_K3C_PD
#define TP_K3C_PD 4         // pieces ahead: T' loads in flight per warp
#endif
#ifndef TP_K3C_MINB
#define TP_K3C_MINB 6       // W = 1: CTAs (8 warps) per SM (40 registers with TP_K3C_RING: 12 warps per sub-partition)
#endif
#ifndef TP_K3C_RING
#define TP_K3C_RING 1       // SINGLE: only the T' values in the prefetch ring (len / Dmin re-read from shared)
#endif
#ifndef TP_K3C_SINGLE
#define TP_K3C_SINGLE 1     // one record buffer per warp (refilled per chunk) vs double-buffered
#endif

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
    const int32_t* run_h;        // pieces per instance
    const int32_t* run_m;        // [n_inst][H] first iteration of each piece
    const uint32_t* run_key;     // [n_inst][H] cell id of each piece
    const long long* piece_d;    // [n_inst][H] Dmin of each piece's tail (ticks; INT64_MAX: none)
    const int32_t* cell_tab;
    const long long* lut_ticks;
    const uint32_t* cell_clamp;
    int32_t n_inst, H, F;
    long long tbt_ticks;
    uint32_t skip;
    int32_t search;
    int32_t* next;               // W = 1: instance counter (count - 1; -1 when idle)
    int32_t* done;               // W = 1: CTAs finished (count - 1)
};

// T += len * t for 64-bit T, t and a 32-bit len (exact while T < 2^64; T_R < 2^58)
__device__ __forceinline__ unsigned long long mad_len(unsigned long long T, unsigned len, unsigned long long t) {
    asm("{\n\t.reg .u32 lo, hi;\n\t"
        "mad.wide.u32 %0, %1, %2, %0;\n\t"
        "mov.b64 {lo, hi}, %0;\n\t"
        "mad.lo.u32 hi, %1, %3, hi;\n\t"
        "mov.b64 %0, {lo, hi};\n\t}"
        : "+l"(T) : "r"(len), "r"((unsigned)t), "r"((unsigned)(t >> 32)));
    return T;
}
// &col[off] as one IMAD.WIDE.U32 (col: this lane's column of the T' table, off: a row's offset)
template <typename TV>
__device__ __forceinline__ const TV* tab_at(const TV* col, unsigned off) {
    const TV* a;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a) : "r"(off), "n"((int)sizeof(TV)), "l"(col));
    return a;
}
// T' table loads through L1 (default: hot cells are shared by many instances, C5 K3c 527 -> 497 us)
// or L2 only (TP_K3C_LDG=0)
#ifndef TP_K3C_LDG
#define TP_K3C_LDG 1
#endif
#ifndef TP_K3C_CARVE
#define TP_K3C_CARVE -1      // preferred shared-memory carveout in percent (-1: the driver's choice)
#endif
template <typename TV>
__device__ __forceinline__ TV lut_load(const TV* a) {
#if TP_K3C_LDG
    return __ldg(a);
#else
    return __ldcg(a);
#endif
}
// the 32-bit table (units of 2^8 ticks): one 32 x 32 -> 64-bit multiply-add
__device__ __forceinline__ unsigned long long mad_len(unsigned long long T, unsigned len, unsigned t) {
    return T + (unsigned long long)len * t;
}

// W warps per instance: warp w walks the pieces [h*w/W, h*(w+1)/W) with a local T_R starting at 0;
// it leaves its total S_w[u] and its Eq. 4 margin M_w[u] = min over its pieces of
// (Dmin - T_local(tail)) (integers, exact); the instance passes at u iff P_w < M_w for every w,
// P_w = S_0 + ... + S_{w-1} (T_R(tail) = P_w + T_local(tail) < Dmin), and the TBT check holds on
// the total.  W = 1 keeps the early exit once every level has failed.  L32: the T' table holds
// uint32 units of 2^8 ticks (model tick_shift = 8) and T_R / Dmin count the same units.
template <int W, bool L32>
__global__ void __launch_bounds__(kWarpsPerCta * 32, W == 1 ? TP_K3C_MINB : 4)
k3_compact(const __grid_constant__ K3cParams p) {
    using TV = typename std::conditional<L32, unsigned, unsigned long long>::type;
    constexpr int IPC = kWarpsPerCta / W;            // instances per CTA
    constexpr int PD = TP_K3C_PD;
    static_assert(32 % PD == 0 && PD <= 16, "prefetch distance divides the chunk");
    __shared__ int4 s_rec[kWarpsPerCta][2][32];       // each warp's staged piece records, double-buffered
    __shared__ long long s_S[W > 1 ? kWarpsPerCta : 1][32], s_M[W > 1 ? kWarpsPerCta : 1][32];
    __shared__ uint32_t s_cm[W > 1 ? kWarpsPerCta : 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = warp / W, w = warp % W;             // instance slot in the CTA, segment
    // the warp's own named barrier for the staged-record hand-offs (a __syncwarp() can be
    // compiled to nothing; see k1_compact.cu Group::sync)
    auto wsync = [&]() { warp_bar(warp + 1); };
    pdl_wait();                                       // K1c / K2 outputs
    const int F = p.F;
    // W = 1: persistent warps, each takes the next instance from a global counter (instances
    // differ a lot in length; a static assignment leaves warps idle behind the longest one of
    // their CTA); W > 1: one instance per W-warp group
    int i = blockIdx.x * IPC + g;
    for (;; ) {
    if constexpr (W == 1) {
        int t = 0;
        if (lane == 0) t = atomicAdd(p.next, 1) + 1;     // next holds count - 1
        i = __shfl_sync(kFull, t, 0);
        if (i >= p.n_inst) break;
    }
    const bool live = i < p.n_inst;
    uint32_t st = 0;
    bool skipped = true;
    if (live) {
        st = p.status[i];
        skipped = (st & p.skip) != 0;
        if (skipped && w == 0 && lane == 0)
            p.level[i] = (st & TP_ST_BAD_INPUT) ? F - 1 : (st & TP_ST_EMPTY) ? 0 : F - 1;
    }
    if (W == 1 && (!live || skipped)) continue;
    const bool work = live && !skipped;               // warp-uniform (same instance for the W warps)
    unsigned long long T = 0;                         // local T_R at the last tail walked (< 2^58)
    long long M = kNoDeadline;                        // Eq. 4 margin (W > 1)
    bool ok = lane < F;                               // W == 1: pass so far
    uint32_t cm = 0;                                  // OR of the pieces' cell clamp masks
    int n = 0;
    if (work) {
        n = p.n[i];
        const int h = p.run_h[i];
        const size_t row = (size_t)i * p.H;
        const int ka = (int)((int64_t)h * w / W), kz = (int)((int64_t)h * (w + 1) / W);
        // this lane's column of the T' table (by cell id; lanes >= F read column F-1 -- ignored)
        const TV* col = reinterpret_cast<const TV*>(p.lut_ticks) + min(lane, F - 1);
        // piece k's record, lane-parallel: {cell id * F, len, Dmin lo, Dmin hi}; padding past kz
        // (len 0, no deadline; the T' row of the chunk's first piece, so every T' load reads a row
        // K2 wrote) walks as a no-op
        int s0 = 0, s1 = 0;
        uint32_t key = 0;
        long long d = kNoDeadline;
        bool v = false;
        auto fetch = [&](int k) {
            v = k < kz;
            if (v) {
                s0 = __ldg(p.run_m + row + k);
                s1 = (k + 1 < h) ? __ldg(p.run_m + row + k + 1) : n + 1;
                key = __ldg(p.run_key + row + k);
                d = __ldg(p.piece_d + row + k);
            }
        };
        auto stage = [&](int4* buf) {
            const int off = (int)(key * (uint32_t)F);
            const int off0 = __shfl_sync(kFull, off, 0);          // lane 0's piece is always real
            buf[lane] = v ? make_int4(off, s1 - s0, (int)(unsigned)d, (int)(d >> 32))
                          : make_int4(off0, 0, -1, 0x7fffffff);
            if (v) cm |= __ldcg(p.cell_clamp + key);
        };
#if TP_K3C_SINGLE
        // one buffer: records of chunk kb staged at its start, then the ring primed and walked
        int4* buf = s_rec[warp][0];
        for (int kb = ka; kb < kz; kb += 32) {
            fetch(kb + lane);
            wsync();                             // the previous chunk's reads of buf are done
            stage(buf);
            wsync();
            const int cnt = min(32, kz - kb);
#if TP_K3C_RING
            // only the T' loads ride in registers; len and Dmin are re-read from the staged record
            // when the piece is walked (a broadcast shared load): 16 registers fewer
            TV rt[PD];
#pragma unroll
            for (int j = 0; j < PD; ++j) rt[j] = lut_load(tab_at(col, (unsigned)buf[j].x));
            auto group = [&](int q0, auto more) {
#pragma unroll
                for (int j = 0; j < PD; ++j) {
                    TV tn = 0;
                    if constexpr (decltype(more)::value) tn = lut_load(tab_at(col, (unsigned)buf[q0 + PD + j].x));
                    const int4 r = buf[q0 + j];
                    const unsigned long long dd = ((unsigned long long)(unsigned)r.w << 32) | (unsigned)r.z;
                    T = mad_len(T, (unsigned)r.y, rt[j]);   // T_R at this piece's tail (Eq. 3)
                    if (W == 1) ok &= T < dd;                 // Eq. 4, strict (Dmin >= 0: unsigned compare)
                    else M = min(M, (long long)dd - (long long)T);
                    if constexpr (decltype(more)::value) rt[j] = tn;
                }
            };
#else
            TV rt[PD];
            unsigned rl[PD];
            unsigned long long rd[PD];
#pragma unroll
            for (int j = 0; j < PD; ++j) {
                const int4 r = buf[j];
                rt[j] = lut_load(tab_at(col, (unsigned)r.x));
                rl[j] = (unsigned)r.y;
                rd[j] = ((unsigned long long)(unsigned)r.w << 32) | (unsigned)r.z;
            }
            auto group = [&](int q0, auto more) {
#pragma unroll
                for (int j = 0; j < PD; ++j) {
                    int4 r;
                    TV tn = 0;
                    if constexpr (decltype(more)::value) {
                        r = buf[q0 + PD + j];         // broadcast: the record PD pieces ahead
                        tn = lut_load(tab_at(col, (unsigned)r.x));
                    }
                    T = mad_len(T, rl[j], rt[j]);     // T_R at this piece's tail (Eq. 3)
                    if (W == 1) ok &= T < rd[j];      // Eq. 4, strict (Dmin >= 0: unsigned compare)
                    else M = min(M, (long long)rd[j] - (long long)T);
                    if constexpr (decltype(more)::value) {
                        rt[j] = tn;
                        rl[j] = (unsigned)r.y;
                        rd[j] = ((unsigned long long)(unsigned)r.w << 32) | (unsigned)r.z;
                    }
                }
            };
#endif
            int q0 = 0;
            for (; q0 + PD < cnt; q0 += PD) group(q0, std::true_type{});
            group(q0, std::false_type{});             // the last group: padding past cnt is a no-op
            if (W == 1 && !__any_sync(kFull, ok)) {  // every level failed: only the clamp OR is left
                for (int k2 = kb + 32 + lane; k2 < kz; k2 += 32) cm |= __ldcg(p.cell_clamp + __ldg(p.run_key + row + k2));
                break;
            }
        }
#else
        int cb = 0;                                   // buffer of the current chunk
        if (ka < kz) {
            fetch(ka + lane);
            stage(s_rec[warp][0]);
            wsync();
        }
        // the next PD pieces in flight: their T' loads issued, len and Dmin in registers
        TV rt[PD];
        unsigned rl[PD];
        unsigned long long rd[PD];
#pragma unroll
        for (int j = 0; j < PD; ++j) {
            const int4 r = s_rec[warp][0][j];
            rt[j] = lut_load(tab_at(col, (unsigned)r.x));
            rl[j] = (unsigned)r.y;
            rd[j] = ((unsigned long long)(unsigned)r.w << 32) | (unsigned)r.z;
        }
        for (int kb = ka; kb < kz; kb += 32, cb ^= 1) {
            const int4* cur = s_rec[warp][cb];
            int4* nxt = s_rec[warp][cb ^ 1];
            const int cnt = min(32, kz - kb);
            fetch(kb + 32 + lane);                    // the next chunk's records, staged at step 32 - PD
            for (int q0 = 0; q0 < 32; q0 += PD) {
                if (q0 >= cnt) break;                 // uniform: the ragged last chunk
                if (q0 == 32 - PD) {
                    wsync();                     // the previous chunk's reads of nxt are done
                    stage(nxt);
                    wsync();
                }
                const int4* ahead = q0 + PD < 32 ? cur + q0 + PD : nxt + (q0 + PD - 32);
#pragma unroll
                for (int j = 0; j < PD; ++j) {
                    const int4 r = ahead[j];          // broadcast: the record PD pieces ahead
                    const TV tn = lut_load(tab_at(col, (unsigned)r.x));
                    T = mad_len(T, rl[j], rt[j]);     // T_R at this piece's tail (Eq. 3)
                    if (W == 1) ok &= T < rd[j];      // Eq. 4, strict (Dmin >= 0: unsigned compare)
                    else M = min(M, (long long)rd[j] - (long long)T);
                    rt[j] = tn;
                    rl[j] = (unsigned)r.y;
                    rd[j] = ((unsigned long long)(unsigned)r.w << 32) | (unsigned)r.z;
                }
            }
            if (W == 1 && !__any_sync(kFull, ok)) {  // every level failed: only the clamp OR is left
                for (int k2 = kb + 64 + lane; k2 < kz; k2 += 32) cm |= __ldcg(p.cell_clamp + __ldg(p.run_key + row + k2));
                break;
            }
        }
#endif
    }
    cm = __reduce_or_sync(kFull, cm);
    if (W > 1) {
        s_S[warp][lane] = (long long)T;
        s_M[warp][lane] = M;
        if (lane == 0) s_cm[warp] = cm;
        __syncthreads();
        if (w != 0 || !work) break;
        long long P = 0;
#pragma unroll
        for (int v = 0; v < W; ++v) {
            ok &= P < s_M[g * W + v][lane];
            P += s_S[g * W + v][lane];
            cm |= s_cm[g * W + v];
        }
        T = (unsigned long long)P;
    }
    ok &= (long long)T <= ((long long)n * p.tbt_ticks) >> (L32 ? 8 : 0);   // TBT: T_R[n] <= n * slo
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
    if constexpr (W > 1) break;
    }
    if constexpr (W == 1) {                           // the last CTA out re-arms the counter
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(p.done, 1) + 1 == (int)gridDim.x - 1) {
                atomicExch(p.next, -1);
                atomicExch(p.done, -1);
            }
        }
    }
}

}  // namespace

int launch_select_compact(const K2Params& w, int32_t n_inst, const int32_t* n, int32_t H, int32_t F,
                          int64_t tbt_ticks, int search, uint32_t skip, int32_t* level, uint32_t* status,
                          cudaStream_t s) {
    if (n_inst == 0) return TP_OK;
    if (!w.cell_tab || !w.end_d || !w.k3_next || F < 1 || F > kMaxF || (search != 0 && search != 1)) return TP_EINVAL;
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
    p.piece_d = w.end_d;
    p.next = w.k3_next;
    p.done = w.k3_done;
    p.n_inst = n_inst;
    p.H = H;
    p.F = F;
    p.tbt_ticks = (long long)tbt_ticks;
    p.skip = skip;
    p.search = search;
    if (w.tick_shift != 0 && w.tick_shift != 8) return TP_EINVAL;
    // warps per instance: enough warps to fill the GPU at small batches (the walk of one instance is
    // a dependent chain of L2 round trips), one per instance at large ones
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static const int w_env = env_warps();
    const int64_t slots = (int64_t)sms * 32;          // resident warps at 8-warp CTAs, 4 per SM
    int W = w_env > 0 ? w_env : (n_inst * 8 <= slots ? 8 : n_inst * 4 <= slots ? 4 : n_inst * 2 <= slots ? 2 : 1);
    auto launch = [&](auto kern, int ipc) {
        int grid = (n_inst + ipc - 1) / ipc;
        if (ipc == kWarpsPerCta) {                    // W = 1: persistent, as many CTAs as fit at once
            static int per_sm[2][64] = {};
            const int li = w.tick_shift == 8;
            if (dev < 64 && per_sm[li][dev] == 0) {
                if (TP_K3C_CARVE >= 0) cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, TP_K3C_CARVE);
                int b = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kWarpsPerCta * 32, 0);
                per_sm[li][dev] = b > 0 ? b : 1;
            }
            grid = std::min(grid, sms * (dev < 64 ? per_sm[li][dev] : 1));
        }
        launch_pdl(kern, dim3(grid), dim3(kWarpsPerCta * 32), 0, s, p);
    };
    const bool l32 = w.tick_shift == 8;
    switch (W) {
        case 8: l32 ? launch(k3_compact<8, true>, 1) : launch(k3_compact<8, false>, 1); break;
        case 4: l32 ? launch(k3_compact<4, true>, 2) : launch(k3_compact<4, false>, 2); break;
        case 2: l32 ? launch(k3_compact<2, true>, 4) : launch(k3_compact<2, false>, 4); break;
        default: l32 ? launch(k3_compact<1, true>, 8) : launch(k3_compact<1, false>, 8); break;
    }
    return cudaPeekAtLastError() == cudaSuccess ? TP_OK : TP_ECUDA;
}

}  // namespace tp
