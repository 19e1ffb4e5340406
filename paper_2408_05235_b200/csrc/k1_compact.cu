// K1c -- the compact path's first kernel: KV usage & batch-size projection (PAPER §4.2, Eq. 1-2,
// P:432-469) with the FIFO admission gate (check 1 + batch cap, §4.3.2, one request at a
// time P:755), fused with what the two later kernels need from it:
//   * pieces + cell claims: M depends on m only through the cell (rank_tp, rank_B[m], rank_KV[m])
//     of the grid row (reading A-7), so m = 1..n is cut into pieces of one cell that also
//     end at every request's last iteration (piece_rules below); first-seen cells are appended to
//     the cell list K2 evaluates;
//   * Eq. 4 per piece: Dmin of the piece's tail = min over the scheduled requests ending
//     there of ceil(fl64(t_dead - t_cur) * 2^40) (reading A-12) -- K3c checks T_R there.
// The B/KV curves never leave the SM unless the caller asks for them (bkv_rows).
//
// One to four WARPS per instance (the CTA-per-instance K1 spends most of its issue slots on
// block-wide phases and barriers at large batches; at small batches a few warps per instance
// shorten its chain of dependent loads): the events go to a per-instance shared histogram, the
// scans and the gate use warp shuffles plus, across the instance's warps, a named barrier and
// shared exchange slots.  Group lane t owns the contiguous segment m in [1 + t*S, 1 + (t+1)*S)
// (S a power of two >= 4); segments are padded by P = 4 words when S/4 is even so that 8
// consecutive lanes' 128-bit accesses fall in distinct bank quads.
#include <algorithm>
#include <cstdlib>

#include "tp_internal.cuh"

namespace tp {
namespace {

constexpr int kWarpsPerCta = 4;
template <int WPI> __host__ __device__ constexpr int cta_warps() { return WPI > kWarpsPerCta ? WPI : kWarpsPerCta; }
constexpr unsigned kFull = 0xffffffffu;

struct SegGeom {
    int S_log2, P, arr;         // segment length 2^S_log2, pad words, ints per array
};

// G group lanes (32 per warp of the instance's group) share the horizon: lane t owns the segment
// m in [1 + t*S, 1 + (t+1)*S), S = 2^k >= 4 with G*S >= H.
SegGeom seg_geom(int H, int G) {
    const int need = (H + G - 1) / G;
    int S = 4, l = 2;
    while (S < need) {
        S <<= 1;
        ++l;
    }
    const int P = ((S / 4) % 2 == 0) ? 4 : 0;
    return {l, P, G * (S + P) + 8};
}

struct K1cParams {
    const tp_inst* inst;
    const int4* req;
    const double* t_dead;
    int32_t n_inst, n_req, H;
    int32_t* B;
    int32_t* KV;
    int32_t bkv_rows;
    int32_t* n;
    int32_t* n_adm;
    uint32_t* status;
    const int32_t* force_adm;
    const uint32_t* lost_mask;
    uint32_t skip;
    int32_t S_log2, P, arr;
    const float* cuts;
    int32_t cut_off[5];
    const uint16_t* rtab;
    int32_t rtab_off[2], rtab_len[2];
    int32_t* run_h;
    int32_t* run_m;
    uint32_t* run_key;
    int32_t* cell_tab;
    uint32_t* cell_list;
    int32_t* cell_count;
    uint32_t* cell_clamp;
    int32_t* end_n;
    long long* end_d;
    int32_t tick_shift;      // Dmin in units of 2^tick_shift ticks (K2Params::tick_shift)
    int32_t* next;           // (unused by K1c; reset with K3c's counters)
    int32_t tab_words;       // k1_packed<true>: 32-bit words of the rank tables staged in shared memory
    int32_t* flag_count;     // k1_packed -> wide fallback hand-over (count - 1)
    int32_t* flag_list;
};

__device__ __forceinline__ uint32_t rank_of(const float* __restrict__ c, int cnt, float x) {
    int lo = 0, hi = cnt;   // number of cuts <= x
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(c + mid) <= x) lo = mid + 1;
        else hi = mid;
    }
    return (uint32_t)lo;
}

__device__ __forceinline__ int warp_max(int v) { return __reduce_max_sync(kFull, v); }

// The WPI warps that own one instance: a named barrier and double-buffered exchange slots in
// shared memory (warp-level values -> every warp of the group sees all WPI of them).
template <int WPI>
struct Group {
    int gw;                     // warp index in the group
    int bar;                    // named barrier id
    long long* xs;              // [2][WPI][4]
    int par = 0;
    // a hardware named barrier even for one warp (warp_bar, tp_internal.cuh)
    __device__ __forceinline__ void sync() const {
        if (WPI == 1) warp_bar(bar);
        else asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(WPI * 32) : "memory");
    }
    // publish 4 warp-level values (lane 0 writes), barrier, return the slot array of this round
    __device__ __forceinline__ const long long* exchange(long long a, long long b, long long c, long long d) {
        if (WPI == 1) return nullptr;
        long long* x = xs + (size_t)par * WPI * 4;
        if ((threadIdx.x & 31) == 0) {
            x[gw * 4 + 0] = a;
            x[gw * 4 + 1] = b;
            x[gw * 4 + 2] = c;
            x[gw * 4 + 3] = d;
        }
        sync();
        par ^= 1;
        return x;
    }
    __device__ __forceinline__ int max(int v) {
        v = warp_max(v);
        if (WPI == 1) return v;
        const long long* x = exchange(v, 0, 0, 0);
        int r = (int)x[0];
#pragma unroll
        for (int k = 1; k < WPI; ++k) r = ::max(r, (int)x[k * 4]);
        return r;
    }
};

// Admission-control mode: the number of queued requests forced in (tp_decide_admit's prefix
// states), or -1 for the FIFO gate.
__device__ __forceinline__ int forced_of(const K1cParams& p, int i, int nq) {
    return p.force_adm ? min(max(p.force_adm[i], 0), nq) : -1;
}

// A piece's cell is marked SEEN in the dense cell table: cell_tab[k] &= 0x7fffffff, a fire-and-
// forget reduction (no L2 round trip on the warp's path, idempotent, and a cell already listed --
// index >= 0 -- keeps its index).  -1 (absent, the launch's memset) becomes kCellSeen; after K1c,
// k1_cells_collect appends every seen cell to the list K2 evaluates and gives it its index.
constexpr int32_t kCellSeen = 0x7fffffff;
__device__ __forceinline__ void claim_cell(const K1cParams& p, uint32_t k) {
    atomicAnd(ptr_at(reinterpret_cast<unsigned*>(p.cell_tab), k), (unsigned)kCellSeen);
}

// piece_rules.  K3c accumulates T_R (Eq. 3) piece by piece and checks Eq. 4 at
// piece tails, so K1c cuts m = 1..n into PIECES: maximal runs of consecutive iterations in one cell
// (rank_tp, rank_B[m], rank_KV[m]) -- the model's value is constant on a piece (reading A-7)
// -- that also end at every end position l (the last iteration of a scheduled request).  No
// admissions happen past m = 1, so B only drops, at l + 1, for the requests ending at l: m - 1 is an
// end position iff B[m] < B[m - 1], and the heads are m = 1 plus every m with key(m) != key(m - 1) or
// B[m] < B[m - 1].  Per instance: run_h = #pieces, run_m / run_key = head m / cell id of each piece,
// end_d = Dmin of the piece's tail (piece_deadlines), end_n = #end positions (statistics).

#ifndef TP_K1_DUNROLL
#define TP_K1_DUNROLL 1
#endif
constexpr int kDUnroll = TP_K1_DUNROLL;
// Eq. 4 per piece: end_d[k] = min over the scheduled requests whose last iteration l is piece k's
// tail of ceil(fl64(t_dead - t_cur) * 2^40) (reading A-12), kNoDeadline where none ends.  The piece
// of l comes from the chunk meta (heads before l's 32-iteration chunk + heads in it up to l, - 1).
// The minima collect in shared memory behind the meta when they fit in `words` 32-bit words from
// `base`, else straight in global memory.
template <int WPI>
__device__ __forceinline__ void piece_deadlines(const K1cParams& p, Group<WPI>& grp, int i, const tp_inst& in,
                                                int64_t rb, int n_sched, int nn, int h, const int2* meta,
                                                long long* base, int words, int gl) {
    constexpr int GL = 32 * WPI;
    if (nn == 0) return;
    const size_t row = (size_t)i * p.H;
    const int C = (nn + 31) >> 5;
    long long* D = base + C;                         // behind meta[C] (8 bytes each)
    const bool sm = 2 * (C + h) <= words;
    grp.sync();                                      // meta written by the whole group
    for (int k = gl; k < h; k += GL) {
        if (sm) D[k] = kNoDeadline;
        else p.end_d[row + k] = kNoDeadline;
    }
    grp.sync();
#pragma unroll kDUnroll
    for (int e = gl; e < n_sched; e += GL) {
        const int64_t j = rb + e;
        const int4 r = __ldg(&p.req[j]);
        const int l = r.z - r.x;                     // 1 <= l <= nn (validated; n = max l)
        const int2 mt = meta[(l - 1) >> 5];
        const int k = mt.y + __popc((unsigned)mt.x & (0xffffffffu >> (31 - ((l - 1) & 31)))) - 1;
        const long long d = slack_ticks(__ldg(&p.t_dead[j]) - in.t_cur, p.tick_shift);
        if (sm) atomicMin(&D[k], d);
        else atomicMin(&p.end_d[row + k], d);
    }
    if (sm) {
        grp.sync();
        for (int k = gl; k < h; k += GL) p.end_d[row + k] = D[k];
    }
}

// One instance, by the WPI warps of group grp (histograms sB / sKV in the group's shared memory).
template <int WPI>
__device__ __forceinline__ void k1_body(const K1cParams& p, const int i, Group<WPI>& grp, int* sB, int* sKV,
                                        const int gl, const int lane) {
    constexpr int GL = 32 * WPI;                       // group lanes
    const int SL = p.S_log2, S = 1 << SL, P = p.P, H = p.H;
    auto ph = [&](int m) { return (m - 1) + P * ((m - 1) >> SL); };   // physical index of m >= 1

    const tp_inst in = p.inst[i];
    const int64_t rb = in.req_begin;
    const int nr = in.n_run, nq = in.n_queue, N = in.N;
    const FastDiv fdN((uint32_t)(N > 0 ? N : 1));
    for (int k = gl * 4; k + 3 < p.arr; k += 4 * GL) {
        *reinterpret_cast<int4*>(sB + k) = make_int4(0, 0, 0, 0);
        *reinterpret_cast<int4*>(sKV + k) = make_int4(0, 0, 0, 0);
    }
    grp.sync();

    // ---- validation (include/tp.h conventions) + running requests -> event histograms ----
    bool bad = N < 1 || in.tp < 1 || (int64_t)in.tp >= kFeatLimit || nr < 0 || nq < 0 || in.kv_cap < 0 ||
               in.max_batch < 0 || rb < 0 || rb + (int64_t)nr + nq > (int64_t)p.n_req;
    int64_t foot = 0;
    int nloc = 0, b1 = 0, kv1 = 0;
    bool lost = false;
    if (!bad) {
        for (int e = gl; e < nr + nq; e += GL) {
            const int4 r = __ldg(&p.req[rb + e]);
            const int64_t l64 = (int64_t)r.z - r.x;
            const bool eb = r.x < 0 || r.y < 1 || r.z < 1 || r.x >= kFeatLimit || r.y >= kFeatLimit || l64 < 1 ||
                            l64 > H || (e >= nr && r.x != 0);
            bad |= eb;
            if (eb) continue;
            const int a = r.x, q = r.y, l = (int)l64, aq = a + q;
            if (p.end_n)   // the deadline list reads t_dead at the end: start its trip to L2 now
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p.t_dead + rb + e));
            foot += (int64_t)fdN.div((uint32_t)(aq + l - 2)) + 1;            // ceil((a+l-1+q)/N)
            if (e < nr) {
                nloc = max(nloc, l);
                lost |= (r.w & TP_REQ_LOST) != 0;
                atomicAdd(&sB[ph(l + 1)], -1);
                const int c1 = (int)fdN.div((uint32_t)(aq - 1));              // ceil(aq / N) - 1
                kv1 += c1 + 1;
                ++b1;
                // first m >= 2 with (aq + m - 2) % N == 0, then every N iterations
                for (int m = 2 + (c1 + 1) * N - aq; m <= l; m += N) atomicAdd(&sKV[ph(m)], 1);
                atomicAdd(&sKV[ph(l + 1)], -((int)fdN.div((uint32_t)(aq + l - 2)) + 1));
            }
        }
    }
    // group totals: flags (bad | lost << 1), footprint, b1 | kv1 << 32 (both < 2^31), max l
    {
        unsigned fl = __ballot_sync(kFull, bad) ? 1u : 0u;
        fl |= __ballot_sync(kFull, lost) ? 2u : 0u;
        for (int o = 16; o; o >>= 1) foot += __shfl_xor_sync(kFull, foot, o);
        b1 = __reduce_add_sync(kFull, b1);
        kv1 = __reduce_add_sync(kFull, kv1);
        nloc = warp_max(nloc);
        if (WPI > 1) {
            const long long* x = grp.exchange(fl, foot, (long long)b1 | ((long long)kv1 << 32), nloc);
            fl = 0;
            foot = 0;
            long long bk = 0;
            nloc = 0;
#pragma unroll
            for (int k = 0; k < WPI; ++k) {
                fl |= (unsigned)x[k * 4];
                foot += x[k * 4 + 1];
                bk += x[k * 4 + 2];
                nloc = max(nloc, (int)x[k * 4 + 3]);
            }
            b1 = (int)(bk & 0xffffffffLL);
            kv1 = (int)(bk >> 32);
        }
        bad = (fl & 1u) || foot >= kFeatLimit;
        lost = (fl & 2u) != 0;
    }
    if (bad) {
        if (p.B) {
            const int lim = p.bkv_rows ? H : 1;
            for (int m = gl; m < lim; m += GL) {
                p.B[(int64_t)i * H + m] = 0;
                p.KV[(int64_t)i * H + m] = 0;
            }
        }
        if (gl == 0) {
            p.n[i] = 0;
            p.n_adm[i] = 0;
            p.status[i] = TP_ST_BAD_INPUT;
            if (p.run_h) p.run_h[i] = 0;
            if (p.end_n) p.end_n[i] = 0;
        }
        return;
    }
    // the m = 1 terms of every running request (index ph(1) = 0 gets no other event)
    grp.sync();
    if (gl == 0) {
        sB[0] += b1;
        sKV[0] += kv1;
    }
    grp.sync();

    // ---- inclusive scans over the lane segments ----
    int* segB = sB + gl * (S + P);
    int* segKV = sKV + gl * (S + P);
    const int lo = 1 + gl * S, hi = min(lo + S, H + 1);    // the lane's valid m (may be empty)
    int kvmax = 0;
    {
        int sb = 0, skv = 0;
        for (int k = 0; k < S; k += 4) {
            const int4 b = *reinterpret_cast<const int4*>(segB + k);
            const int4 v = *reinterpret_cast<const int4*>(segKV + k);
            sb += b.x + b.y + b.z + b.w;
            skv += v.x + v.y + v.z + v.w;
        }
        int xb = sb, xkv = skv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int yb = __shfl_up_sync(kFull, xb, o), ykv = __shfl_up_sync(kFull, xkv, o);
            if (lane >= o) {
                xb += yb;
                xkv += ykv;
            }
        }
        int pb = xb - sb, pkv = xkv - skv;
        if (WPI > 1) {          // add the totals of the group's earlier warps
            const long long* x = grp.exchange(__shfl_sync(kFull, xb, 31), __shfl_sync(kFull, xkv, 31), 0, 0);
#pragma unroll
            for (int k = 0; k < WPI; ++k)
                if (k < grp.gw) {
                    pb += (int)x[k * 4];
                    pkv += (int)x[k * 4 + 1];
                }
        }
        for (int k = 0; k < S; k += 4) {
            int4 b = *reinterpret_cast<const int4*>(segB + k);
            int4 v = *reinterpret_cast<const int4*>(segKV + k);
            b.x += pb; b.y += b.x; b.z += b.y; b.w += b.z;
            v.x += pkv; v.y += v.x; v.z += v.y; v.w += v.z;
            pb = b.w;
            pkv = v.w;
            *reinterpret_cast<int4*>(segB + k) = b;
            *reinterpret_cast<int4*>(segKV + k) = v;
            const int m = lo + k;   // positions past H are padding (never outputs)
            kvmax = max(kvmax, max(max(m <= H ? v.x : 0, m + 1 <= H ? v.y : 0),
                                   max(m + 2 <= H ? v.z : 0, m + 3 <= H ? v.w : 0)));
        }
    }
    int kvb = grp.max(kvmax);          // (its barrier also publishes the scan)
    uint32_t st = kvb > in.kv_cap ? TP_ST_KV_OVER : 0u;

    // ---- FIFO gate: queued c admitted iff B[1]+1 <= max_batch and max_m KV + KV_c <= kv_cap ----
    // One candidate at a time, lane-strided over its window m = 1..l_c.  Only the window
    // needs checking: if max_m KV[m] > kv_cap already (KV_OVER) every candidate fails, and every
    // admission keeps max_m KV[m] <= kv_cap, so past l_c (where KV_c = 0) the check always holds.
    int n_adm = 0;
    const int forced = p.force_adm ? min(max(p.force_adm[i], 0), nq) : -1;
    const uint32_t lmask = p.lost_mask ? p.lost_mask[i] : 0u;
    const int ncand = forced >= 0 ? forced : nq;
    if (WPI == 1) grp.sync();
    if (forced < 0 && ncand > 0 && (st & TP_ST_KV_OVER)) {
        st |= TP_ST_QUEUE_BLOCKED;
    } else {
        int B1 = sB[0];                                  // B[1] (uniform)
        for (int c = 0; c < ncand; ++c) {
            const int4 r = __ldg(&p.req[rb + nr + c]);  // a = 0 (validated)
            const int q = r.y, lc = r.z;
            // kvb: an upper bound of max_m KV[m] (exact after the scan).  KV_c[m] <= KV_c[l_c] on
            // the window, so kvb + KV_c[l_c] <= kv_cap admits without scanning the window
            const int kvc_top = (int)fdN.div((uint32_t)(lc + q - 2)) + 1;
            if (forced < 0) {
                bool admit = B1 + 1 <= in.max_batch;
                if (admit && kvb + kvc_top > in.kv_cap) {
                    int mx = 0;
#pragma unroll 4
                    for (int m = 1 + gl; m <= lc; m += GL)   // Eq. 1: KV_c[m] = ceil((m - 1 + q) / N)
                        mx = max(mx, sKV[ph(m)] + (int)fdN.div((uint32_t)(m + q - 2)) + 1);
                    mx = grp.max(mx);
                    admit = mx <= in.kv_cap;
                    kvb = max(kvb, mx);              // past the window KV is unchanged (<= kvb)
                } else {
                    kvb += kvc_top;
                }
                if (!admit) {
                    st |= TP_ST_QUEUE_BLOCKED;
                    break;
                }
            } else {
                kvb += kvc_top;
            }
#pragma unroll 4
            for (int m = 1 + gl; m <= lc; m += GL) {
                const int pi = ph(m);
                sKV[pi] += (int)fdN.div((uint32_t)(m + q - 2)) + 1;
                sB[pi] += 1;
            }
            grp.sync();
            ++B1;
            ++n_adm;
            nloc = max(nloc, lc);
            lost |= (r.w & TP_REQ_LOST) || (c < 32 && ((lmask >> c) & 1u));
        }
    }
    if (forced >= 0 && forced < nq) st |= TP_ST_QUEUE_BLOCKED;
    const int n = nloc;                              // group-uniform (admitted l's are uniform)
    if (n == 0) st |= TP_ST_EMPTY;
    else if (lost) st |= TP_ST_BYPASS_LOST;
    grp.sync();

    if (p.B) {
        int* Bo = p.B + (int64_t)i * H;
        int* Ko = p.KV + (int64_t)i * H;
        if (!p.bkv_rows) {
            if (gl == 0) {
                Bo[0] = sB[0];
                Ko[0] = sKV[0];
            }
        } else if ((H & 3) == 0) {   // rows 16-byte aligned: 128-bit stores (groups never straddle)
            for (int v = gl; v < (H >> 2); v += GL) {
                const int m = 4 * v + 1;
                reinterpret_cast<int4*>(Bo)[v] = *reinterpret_cast<const int4*>(sB + ph(m));
                reinterpret_cast<int4*>(Ko)[v] = *reinterpret_cast<const int4*>(sKV + ph(m));
            }
        } else {
            for (int m = 1 + gl; m <= H; m += GL) {
                Bo[m - 1] = sB[ph(m)];
                Ko[m - 1] = sKV[ph(m)];
            }
        }
    }
    if (gl == 0) {
        p.n[i] = n;
        p.n_adm[i] = n_adm;
        p.status[i] = st;
    }
    const int nn = (st & p.skip) ? 0 : n;    // iterations K2 / K3 evaluate
    const unsigned ltm = (1u << lane) - 1u;
    const size_t row = (size_t)i * H;

    // ---- pieces over m = 1..nn (see piece_rules below), first-seen cells claimed ----
    // Group-strided over m (warp gw takes the 32 iterations m0 + 32 gw + lane, i.e. 32-chunk
    // c = (m0 - 1) / 32 + gw): key, B, head flag, ballot; records written straight from the
    // compaction; across warps the first / last (key, B) and head counts go through the exchange,
    // whose barrier also orders every histogram read of the step before the meta writes.
    const int nB = p.cut_off[2] - p.cut_off[1], nKV = p.cut_off[3] - p.cut_off[2];
    const int lB = p.rtab_len[0], lKV = p.rtab_len[1];
    const uint16_t* tB = p.rtab + p.rtab_off[0];
    const uint16_t* tKV = p.rtab + p.rtab_off[1];
    const uint32_t rtp = rank_of(p.cuts + p.cut_off[0], p.cut_off[1] - p.cut_off[0], (float)in.tp);
    const uint32_t nk1 = (uint32_t)nKV + 1;
    const uint32_t cell_base = rtp * (uint32_t)(nB + 1) * nk1;
    int2* meta = reinterpret_cast<int2*>(sB);        // [chunk] (head mask, heads before the chunk)
    int h = 0, ends = 0;
    uint32_t kcarry = 0xffffffffu;                   // key / B of m0 - 1 (m = 1 always starts a piece)
    int bcarry = 0;
    for (int m0 = 1; m0 <= nn; m0 += GL) {
        const int m = m0 + gl;
        uint32_t k = 0;
        int b = 0;
        if (m <= nn) {
            const int pi = ph(m);
            b = sB[pi];
            const int kv = sKV[pi];
            const uint32_t rbk = b < lB ? __ldg(tB + b) : rank_of(p.cuts + p.cut_off[1], nB, (float)b);
            const uint32_t rkv = kv < lKV ? __ldg(tKV + kv) : rank_of(p.cuts + p.cut_off[2], nKV, (float)kv);
            k = cell_base + rbk * nk1 + rkv;
        }
        const uint32_t pk = __shfl_up_sync(kFull, k, 1);
        const int pb = __shfl_up_sync(kFull, b, 1);
        const uint32_t kfirst = __shfl_sync(kFull, k, 0), klast = __shfl_sync(kFull, k, 31);
        const int bfirst = __shfl_sync(kFull, b, 0), blast = __shfl_sync(kFull, b, 31);
        const bool live = m <= nn;
        const bool head_rest = lane > 0 && live && (k != pk || b < pb);     // lanes 1..31
        const unsigned mrest = __ballot_sync(kFull, head_rest);
        const unsigned erest = __ballot_sync(kFull, lane > 0 && live && b < pb);   // m - 1 is an end
        int before = 0, tot = 0, etot = 0;           // heads / ends of this step in earlier warps, all
        bool head0, end0;                            // this warp's lane-0 flags (vs the previous chunk)
        if (WPI == 1) {
            head0 = m0 <= nn && (kfirst != kcarry || bfirst < bcarry);
            end0 = m0 <= nn && bfirst < bcarry;
            tot = __popc(mrest) + head0;
            etot = __popc(erest) + end0;
            kcarry = klast;
            bcarry = blast;
        } else {
            const long long* x = grp.exchange((long long)kfirst | ((long long)klast << 32),
                                              (long long)(unsigned)bfirst | ((long long)blast << 32),
                                              __popc(mrest), __popc(erest));
            uint32_t pkl = kcarry;
            int pbl = bcarry;
            head0 = end0 = false;
#pragma unroll
            for (int v = 0; v < WPI; ++v) {
                const uint32_t kf = (uint32_t)x[v * 4], kl = (uint32_t)(x[v * 4] >> 32);
                const int bf = (int)(uint32_t)x[v * 4 + 1], bl = (int)(x[v * 4 + 1] >> 32);
                const bool lv = m0 + 32 * v <= nn;
                const bool ev = lv && bf < pbl, hv = lv && (kf != pkl || bf < pbl);
                if (v < grp.gw) before += (int)x[v * 4 + 2] + hv;
                if (v == grp.gw) {
                    head0 = hv;
                    end0 = ev;
                }
                tot += (int)x[v * 4 + 2] + hv;
                etot += (int)x[v * 4 + 3] + ev;
                pkl = kl;
                pbl = bl;
            }
            kcarry = pkl;
            bcarry = pbl;
        }
        const unsigned mask = mrest | (head0 ? 1u : 0u);
        if (lane == 0 ? head0 : head_rest) {
            const int pos = h + before + __popc(mask & ltm);
            p.run_m[row + pos] = m;
            p.run_key[row + pos] = k;
            claim_cell(p, k);
        }
        if (lane == 0 && m <= nn) meta[(m - 1) >> 5] = make_int2((int)mask, h + before);
        h += tot;
        ends += etot;
    }
    if (gl == 0) {
        p.run_h[i] = h;
        p.end_n[i] = nn > 0 ? ends + 1 : 0;          // + m = nn, always an end
    }
    piece_deadlines<WPI>(p, grp, i, in, rb, nr + n_adm, nn, h, meta, reinterpret_cast<long long*>(sB),
                         2 * p.arr, gl);
}

// ---------------------------------------------------------------------------------------------
// K1c, packed (large batches, one warp per instance): the two histograms in ONE int32 array,
// value = B[m] * 2^16 + KV[m] -- exact whenever B < 2^15 and KV < 2^16, which the footprint check
// certifies per instance (B <= R + Q, KV <= the sum of the requests' final block counts); the
// difference-array events and the scan then work on the packed words unchanged (two's-complement
// sums), and one atomic carries both end-of-request events.  Half the shared memory of k1_compact<1>
// (more resident warps: this kernel is latency-bound) and half the scan work.  Run records are
// written straight from the ballot compaction (consecutive positions per step: coalesced); the
// Eq. 4 table is built in windows of the histogram space.  Instances the check rejects are handed
// to k1_compact<1, true> through the flag list.
#ifndef TP_K1P_WARPS
// warps (instances in flight) per CTA (named barriers 1..15).  12: three CTAs of 12 warps at 48
// registers fill each SM sub-partition's 16 K registers with 9 warps (36 per SM); 13 or 14 put
// 4 warps of every CTA on sub-partition 0, so only two CTAs fit (26-28 warps)
#define TP_K1P_WARPS 12
#endif
#ifndef TP_K1P_RTP
#define TP_K1P_RTP 1         // engine-size ranks from a per-CTA table (0: a binary search per instance)
#endif
#ifndef TP_K1P_REQPF
#define TP_K1P_REQPF 1       // request loop: the lane's next record loaded one iteration ahead
#endif
#ifndef TP_K1P_EQ4PF
#define TP_K1P_EQ4PF 1       // Eq. 4 pass: the lane's first record + deadline loaded before the piece passes
#endif
#ifndef TP_K1P_ST
#define TP_K1P_ST 1          // rank tables staged in shared memory when they fit (0: read through L1)
#endif
#ifndef TP_K1P_LINEAR
#define TP_K1P_LINEAR 1      // unpadded histogram, scans over the S2 lane segments
#endif
#ifndef TP_K1P_BALB
#define TP_K1P_BALB 1        // pass B records distributed round-robin over the lanes
#endif
#ifndef TP_K1P_ZDIRTY
#define TP_K1P_ZDIRTY 1      // clear only the prefix of the histogram the previous instance wrote
#endif
#ifndef TP_K1P_MERGE
#define TP_K1P_MERGE 1       // scan + pass A in one pass when no FIFO candidate is left for the gate
#endif
#ifndef TP_K1P_BATCHQ
#define TP_K1P_BATCHQ 1      // the bound-covered prefix of the FIFO queue admitted as events before the scan
#endif
#ifndef TP_K1P_EQ4B
#define TP_K1P_EQ4B 1        // Eq. 4 pass: records per lane loaded together (1: one ahead)
#endif
#ifndef TP_K1P_MAXREG
#define TP_K1P_MAXREG 48     // > 0: register cap instead of the CTAs-per-SM launch bound (48 x 42 warps fill the file)
#endif
#ifndef TP_K1P_MINB
#define TP_K1P_MINB 3        // CTAs per SM when TP_K1P_MAXREG = 0 (3 x (12 x 4.6 KB + 9 KB of tables) at H = 1024)
#endif

// one warp's named barrier (see Group::sync); the id is a register (k1_packed uses up to 15 of them
// anyway: one per warp of its CTA), a switch over immediate ids costs ~10 instructions per barrier
#define K1P_SYNC() asm volatile("bar.sync %0, 32;" ::"r"(w + 1) : "memory")
// +1 at every m = m1, m1 + N, ... <= l (the block increments of one request, Eq. 1) in the padded
// layout ph(m) = m - 1 + P * ((m - 1) >> SL); when N is a multiple of the segment length 2^SL the
// physical stride is the constant N + P * N / 2^SL
__device__ __forceinline__ void block_events(int* sv, int m1, int l, int N, int SL, int P) {
    if (m1 > l) return;
    if ((N & ((1 << SL) - 1)) == 0) {
        const int step = N + P * (N >> SL);
        int pi = (m1 - 1) + P * ((m1 - 1) >> SL);
        #pragma unroll 1
        for (int m = m1; m <= l; m += N, pi += step) atomicAdd(&sv[pi], 1);
    } else {
        #pragma unroll 1
        for (int m = m1; m <= l; m += N) atomicAdd(&sv[(m - 1) + P * ((m - 1) >> SL)], 1);
    }
}
// ST: the B / KV rank tables staged in shared memory (p.tab_words 32-bit words in front of the
// warps' histograms; every lookup an LDS), else read through L1 from global memory.  Persistent:
// the CTAs that fit at once, warp w of CTA b takes instances b * wpb + w, + gridDim.x * wpb, ...
template <bool ST>
#if TP_K1P_MAXREG
__global__ void __maxnreg__(TP_K1P_MAXREG)
#else
__global__ void __launch_bounds__(TP_K1P_WARPS * 32, TP_K1P_MINB)
#endif
k1_packed(const __grid_constant__ K1cParams p) {
    extern __shared__ __align__(16) int smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = (int)(blockDim.x >> 5);
    int* sv = smem + (ST ? p.tab_words : 0) + (size_t)w * p.arr;
    const int lB1 = p.rtab_len[0] - 1, lKV1 = p.rtab_len[1] - 1;   // tables end past the last cut
    const uint16_t* tB;
    const uint16_t* tKV;
    if (lane == 0 && blockIdx.x * wpb + w < p.n_inst) {   // the first instance's request table -> L2
        const int4 f = __ldg(reinterpret_cast<const int4*>(p.inst + blockIdx.x * wpb + w) + 1);
        if (f.y > 0 && f.z >= 0 && f.x >= 0 && (int64_t)f.x + f.y + f.z <= (int64_t)p.n_req)
            prefetch_l2_bulk(p.req + f.x, (uint32_t)(f.y + f.z) * 16u);
    }
    // rank of every engine size tp < 64 among the tp cuts (one binary search per CTA, not per instance)
    __shared__ uint16_t s_rtp[64];
    if (threadIdx.x < 64) s_rtp[threadIdx.x] = (uint16_t)rank_of(p.cuts + p.cut_off[0], p.cut_off[1] - p.cut_off[0],
                                                                 (float)threadIdx.x);
    if constexpr (ST) {
        for (int k = threadIdx.x; k < p.tab_words; k += blockDim.x)
            smem[k] = __ldg(reinterpret_cast<const int*>(p.rtab) + k);
        __syncthreads();
        tB = reinterpret_cast<const uint16_t*>(smem) + p.rtab_off[0];
        tKV = reinterpret_cast<const uint16_t*>(smem) + p.rtab_off[1];
    } else {
        __syncthreads();
        tB = p.rtab + p.rtab_off[0];
        tKV = p.rtab + p.rtab_off[1];
    }
    // TP_K1P_LINEAR: the histogram is unpadded (ph(m) = m - 1); every 128-bit pass walks the
    // S2-word lane segments, S2 / 4 odd where possible, so 8 consecutive lanes hit 8 distinct
    // 16-byte bank groups (the padded layout made the S2 passes 2-6-way conflicted)
    const int SL = p.S_log2, S = 1 << SL, P = TP_K1P_LINEAR ? 0 : p.P, H = p.H;
    auto ph = [&](int m) { return (m - 1) + P * ((m - 1) >> SL); };   // physical index of m >= 1
    int zhi = p.arr;                                  // words of sv to clear for the next instance
#pragma unroll 1
    for (int i = blockIdx.x * wpb + w; i < p.n_inst; i += gridDim.x * wpb) {
    K1P_SYNC();                                       // the previous instance's reads of sv are done

    const tp_inst in = p.inst[i];
    const int64_t rb = in.req_begin;
    const int nr = in.n_run, nq = in.n_queue, N = in.N;
    const FastDiv fdN((uint32_t)(N > 0 ? N : 1));
    // one request's Eq. 1 events: its block increments and the end event at l + 1
    auto req_events = [&](int m1, int l, int kv_end) {
        block_events(sv, m1, l, N, SL, P);
        atomicAdd(&sv[ph(l + 1)], -(65536 + kv_end));                           // B -1 and KV -kv_end
    };
    // the warp's next instance: {req_begin, n_run, n_queue, N}, for the L2 prefetch of its request
    // table below (its loads are then L2 hits instead of HBM round trips)
    const int inext = i + gridDim.x * wpb;
    const bool first = i == blockIdx.x * wpb + w;
    int4 nx = make_int4(0, 0, 0, 0);
    if (lane == 0 && inext < p.n_inst) nx = __ldg(reinterpret_cast<const int4*>(p.inst + inext) + 1);
    #pragma unroll 1
    for (int k = lane * 4; k + 3 < zhi; k += 128) *reinterpret_cast<int4*>(sv + k) = make_int4(0, 0, 0, 0);
    K1P_SYNC();

    bool bad = N < 1 || in.tp < 1 || (int64_t)in.tp >= kFeatLimit || nr < 0 || nq < 0 || in.kv_cap < 0 ||
               in.max_batch < 0 || rb < 0 || rb + (int64_t)nr + nq > (int64_t)p.n_req;
    int64_t foot = 0;
    int nloc = 0, b1 = 0, kv1 = 0;
    bool lost = false;
    if (!bad) {
        const int ne = nr + nq;
#if TP_K1P_REQPF
        // the next record of this lane is loaded before the current one's events (one load in flight
        // behind the shared atomics instead of a full round trip per iteration)
        int4 rn = lane < ne ? __ldg(&p.req[rb + lane]) : make_int4(0, 0, 0, 0);
#if TP_K1P_REQPF > 1
        int4 rn2 = lane + 32 < ne ? __ldg(&p.req[rb + lane + 32]) : make_int4(0, 0, 0, 0);
#endif
#endif
        #pragma unroll 1
        for (int e = lane; e < ne; e += 32) {
#if TP_K1P_REQPF
            const int4 r = rn;
#if TP_K1P_REQPF > 1
            rn = rn2;
            if (e + 64 < ne) rn2 = __ldg(&p.req[rb + e + 64]);
#else
            if (e + 32 < ne) rn = __ldg(&p.req[rb + e + 32]);
#endif
#else
            const int4 r = __ldg(&p.req[rb + e]);
#endif
            const int64_t l64 = (int64_t)r.z - r.x;
            const bool eb = r.x < 0 || r.y < 1 || r.z < 1 || r.x >= kFeatLimit || r.y >= kFeatLimit || l64 < 1 ||
                            l64 > H || (e >= nr && r.x != 0);
            bad |= eb;
            if (eb) continue;
            const int a = r.x, q = r.y, l = (int)l64, aq = a + q;
            // the warp's later instances had their deadlines bulk-prefetched by the previous one
            if (first) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.t_dead + rb + e));
            const int kv_end = (int)fdN.div((uint32_t)(aq + l - 2)) + 1;           // ceil((a+l-1+q)/N)
            foot += kv_end;
            if (e < nr) {
                nloc = max(nloc, l);
                lost |= (r.w & TP_REQ_LOST) != 0;
                const int c1 = (int)fdN.div((uint32_t)(aq - 1));                    // ceil(aq / N) - 1
                kv1 += c1 + 1;
                ++b1;
                req_events(2 + (c1 + 1) * N - aq, l, kv_end);
            }
        }
    }
    bad = __any_sync(kFull, bad);
    for (int o = 16; o; o >>= 1) foot += __shfl_xor_sync(kFull, foot, o);
    b1 = __reduce_add_sync(kFull, b1);
    kv1 = __reduce_add_sync(kFull, kv1);
    nloc = warp_max(nloc);
    lost = __any_sync(kFull, lost);
    bad = bad || foot >= kFeatLimit;
    if (!bad && (nr + nq >= 32768 || foot >= 65536)) {       // does not fit the packed words
        if (lane == 0) p.flag_list[atomicAdd(p.flag_count, 1) + 1] = i;   // flag_count holds count - 1
        zhi = p.arr;
        continue;
    }
    if (bad) {
        if (p.B) {
            const int lim = p.bkv_rows ? H : 1;
            #pragma unroll 1
            for (int m = lane; m < lim; m += 32) {
                p.B[(int64_t)i * H + m] = 0;
                p.KV[(int64_t)i * H + m] = 0;
            }
        }
        if (lane == 0) {
            p.n[i] = 0;
            p.n_adm[i] = 0;
            p.status[i] = TP_ST_BAD_INPUT;
            if (p.run_h) p.run_h[i] = 0;
            if (p.end_n) p.end_n[i] = 0;
        }
        zhi = p.arr;
        continue;
    }
    // Whole-queue admission: when the footprint of running + queued fits the capacity and the
    // whole queue fits the batch cap, every FIFO candidate passes check 1 -- for any admitted
    // prefix, max_m KV[m] <= sum of the requests' final block counts = foot <= kv_cap, and
    // B[1] + c <= b1 + nq <= max_batch -- so the gate admits the whole queue: its requests go into
    // the histogram with the running ones (one scan, no per-candidate window passes).  Same
    // result as the one-at-a-time gate below, which handles every other case.
    const bool allq = nq > 0 && forced_of(p, i, nq) < 0 && foot <= in.kv_cap && b1 + nq <= in.max_batch;
    if (allq) {
        int bq = 0, kvq = 0, lq = 0;
        bool lostq = false;
        #pragma unroll 1
        for (int e = nr + lane; e < nr + nq; e += 32) {
            const int4 r = __ldg(&p.req[rb + e]);     // a = 0 (validated)
            const int q = r.y, l = r.z;
            const int kv_end = (int)fdN.div((uint32_t)(q + l - 2)) + 1;
            const int c1 = (int)fdN.div((uint32_t)(q - 1));
            kvq += c1 + 1;
            ++bq;
            lq = max(lq, l);
            lostq |= (r.w & TP_REQ_LOST) != 0;
            req_events(2 + (c1 + 1) * N - q, l, kv_end);
        }
        b1 += __reduce_add_sync(kFull, bq);
        kv1 += __reduce_add_sync(kFull, kvq);
        nloc = max(nloc, warp_max(lq));
        lost |= __any_sync(kFull, lostq);
    }
    K1P_SYNC();
    if (lane == 0) sv[0] += b1 * 65536 + kv1;     // the m = 1 terms (index 0 gets no other event)
    K1P_SYNC();

    // piece-pass segment length S2 for n iterations: a multiple of 4 (odd multiples preferred:
    // conflict-free 128-bit accesses at lane stride S2), so each lane's segment starts 4-aligned
    // and every 4-iteration batch is one aligned int4 (segments of the padded layout are
    // multiples of 4 long); 32 S2 <= arr for n <= H
    auto s2_of = [](int nn) {
        int S2 = (((nn + 31) >> 5) + 3) & ~3;
        if ((S2 & 4) == 0 && 32 * (S2 - 4) < nn && S2 + 4 <= 32) S2 += 4;
        return S2;
    };
    // ---- inclusive scan of the packed words over the lane segments ----
    // (write = false: only the lane's max of KV, the array is left as it is)
#if TP_K1P_LINEAR
    // over the S2 segments of min(n + 1, H) iterations: every event is at m <= n + 1, and the
    // words past the segments are 0 (nothing was written there)
    auto scan = [&](bool write) {
        const int S2s = s2_of(min(nloc + 1, H));
        int* const seg = sv + lane * S2s;
        int kvm = 0, sum = 0;
        #pragma unroll 1
        for (int k = 0; k < S2s; k += 4) {
            const int4 v = *reinterpret_cast<const int4*>(seg + k);
            sum += v.x + v.y + v.z + v.w;
        }
        int x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        int pre = x - sum;
        #pragma unroll 1
        for (int k = 0; k < S2s; k += 4) {
            int4 v = *reinterpret_cast<const int4*>(seg + k);
            v.x += pre; v.y += v.x; v.z += v.y; v.w += v.z;
            pre = v.w;
            if (write) *reinterpret_cast<int4*>(seg + k) = v;
            // KV[m] = 0 past every request's last iteration, so positions past H need no mask
            kvm = max(kvm, max(max(v.x & 0xFFFF, v.y & 0xFFFF), max(v.z & 0xFFFF, v.w & 0xFFFF)));
        }
        return kvm;
    };
#else
    int* seg = sv + lane * (S + P);
    auto scan = [&](bool write) {
        int kvm = 0, sum = 0;
        #pragma unroll 1
        for (int k = 0; k < S; k += 4) {
            const int4 v = *reinterpret_cast<const int4*>(seg + k);
            sum += v.x + v.y + v.z + v.w;
        }
        int x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        int pre = x - sum;
        #pragma unroll 1
        for (int k = 0; k < S; k += 4) {
            int4 v = *reinterpret_cast<const int4*>(seg + k);
            v.x += pre; v.y += v.x; v.z += v.y; v.w += v.z;
            pre = v.w;
            if (write) *reinterpret_cast<int4*>(seg + k) = v;
            // KV[m] = 0 past every request's last iteration, so positions past H need no mask
            kvm = max(kvm, max(max(v.x & 0xFFFF, v.y & 0xFFFF), max(v.z & 0xFFFF, v.w & 0xFFFF)));
        }
        return kvm;
    };
#endif
    const int forced = forced_of(p, i, nq);
    const uint32_t lmask = p.lost_mask ? p.lost_mask[i] : 0u;
    int c0 = 0;                                    // candidates admitted by the bound below
    int kvb0 = -1;                                 // max_m KV[m] of the running set (bound prefix)
#if TP_K1P_BATCHQ
    // Bound prefix of the FIFO gate: with kvb0 = max_m KV[m] of the running set, candidate c is
    // admitted by check 1 whenever kvb0 + sum_{c' <= c} ceil((q_c' + l_c' - 1) / N) <= kv_cap and
    // B[1] + c + 1 <= max_batch (each admitted request adds at most its final block count at any
    // m), so that prefix of the queue is admitted exactly as the one-at-a-time gate admits it and
    // goes into the difference array as events (one read-only scan instead of a per-iteration add
    // pass per candidate); the gate below continues at the first candidate the bound does not cover.
    if (!allq && nq > 0 && forced < 0) {
        kvb0 = warp_max(scan(false));
        if (kvb0 <= in.kv_cap) {
            const bool has = lane < nq;
            const int4 r = has ? __ldg(&p.req[rb + nr + lane]) : make_int4(0, 1, 1, 0);   // a = 0 (validated)
            const int q = r.y, l = r.z;
            const int top = has ? (int)fdN.div((uint32_t)(q + l - 2)) + 1 : 0;
            int cum = top;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(kFull, cum, o);
                if (lane >= o) cum += y;
            }
            const bool okc = has && (int64_t)kvb0 + cum <= in.kv_cap && b1 + lane + 1 <= in.max_batch;
            const uint32_t nok = ~__ballot_sync(kFull, okc);
            c0 = nok ? __ffs(nok) - 1 : 32;
            if (c0 > 0) {
                K1P_SYNC();                            // every lane's read-only scan is done
                const bool adm = lane < c0;
                if (adm) {
                    const int c1 = (int)fdN.div((uint32_t)(q - 1));
                    req_events(2 + (c1 + 1) * N - q, l, top);
                    atomicAdd(&sv[0], 65536 + c1 + 1);
                }
                nloc = max(nloc, warp_max(adm ? l : 0));
                lost |= __any_sync(kFull, adm && ((r.w & TP_REQ_LOST) || ((lmask >> lane) & 1u)));
                K1P_SYNC();
            }
        }
    }
#endif
    // cell key of a histogram word (b < 2^15, kv < 2^16 here, the packed check: the clamped table
    // lookups are exact) and the piece-pass segment length S2 for n iterations: a multiple of 4
    // (odd multiples preferred: conflict-free 128-bit accesses at lane stride S2), so each lane's
    // segment starts 4-aligned and every 4-iteration batch is one aligned int4 of the padded layout
    // (segments of the scan layout are multiples of 4 long)
    const uint32_t nk1 = (uint32_t)(p.cut_off[3] - p.cut_off[2]) + 1;
    auto key_of = [&](int v) -> uint32_t {
        if constexpr (ST) return (uint32_t)tB[min(v >> 16, lB1)] * nk1 + tKV[min(v & 0xFFFF, lKV1)];
        return (uint32_t)__ldg(ptr_at(tB, (unsigned)min(v >> 16, lB1))) * nk1 +
               __ldg(ptr_at(tKV, (unsigned)min(v & 0xFFFF, lKV1)));
    };
    // Merged scan + pass A: when no FIFO candidate is left for the gate below (no queue, the whole
    // queue admitted, the bound prefix covering it, or the queue blocked by KV_OVER), n is final
    // before the scan, so the scan runs over the piece-pass segments (lane t: m in
    // [1 + t S2, (t+1) S2], n <= 1024) and its second pass computes the keys and head / end flags
    // of pass A on the scanned words in registers: one read + write of each word instead of two,
    // and the neighbour's last word is the lane's exclusive prefix (no shared read).  Values past n
    // are 0 (every request has ended), so the KV max needs no mask.  Not with full B/KV rows out.
    int kvmax = 0, v1 = 0;                         // v1: the word of m = 1 (merged)
    uint32_t mmask = 0;                            // merged: the lane's head mask and end count
    int me = 0;
#if TP_K1P_MERGE
    const bool merged = !(p.B && p.bkv_rows) && s2_of(nloc) <= 32 &&
                        (nq == 0 || allq || (forced < 0 && (kvb0 > in.kv_cap || c0 >= nq)));
#else
    const bool merged = false;
#endif
    if (merged) {
        const int S2 = s2_of(nloc);
        const int mlo = 1 + lane * S2, mhi = min(mlo + S2 - 1, nloc);   // empty when mlo > n
        int sum = 0;
        #pragma unroll 1
        for (int m0 = mlo; m0 <= mhi; m0 += 4) {
            const int4 v = *reinterpret_cast<const int4*>(sv + ph(m0));
            sum += v.x + v.y + v.z + v.w;
        }
        int x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        int pre = x - sum;                         // the word of mlo - 1
        uint32_t pk = 0xffffffffu;                 // key / B of m - 1 (m = 1 always starts a piece)
        int pb = 0;
        if (mlo >= 2 && mlo <= nloc) {
            pb = pre >> 16;
            pk = key_of(pre);
        }
        #pragma unroll 1
        for (int m0 = mlo; m0 <= mhi; m0 += 4) {
            int4* const q = reinterpret_cast<int4*>(sv + ph(m0));
            int4 v = *q;
            v.x += pre; v.y += v.x; v.z += v.y; v.w += v.z;
            pre = v.w;
            kvmax = max(kvmax, max(max(v.x & 0xFFFF, v.y & 0xFFFF), max(v.z & 0xFFFF, v.w & 0xFFFF)));
            if (m0 == 1) v1 = v.x;
            const uint32_t bit = 1u << (m0 - mlo);
            auto flag = [&](int& w, uint32_t bu, bool live) {   // as pass A below
                const uint32_t k = key_of(w);
                const int b = w >> 16;
                const bool endp = live && b < pb;
                const bool head = live && (k != pk || endp);
                mmask |= head ? bu : 0u;
                me += endp;
                w = (int)k;
                pk = k;
                pb = b;
            };
            flag(v.x, bit, true);
            flag(v.y, bit << 1, m0 + 1 <= mhi);
            flag(v.z, bit << 2, m0 + 2 <= mhi);
            flag(v.w, bit << 3, m0 + 3 <= mhi);
            *q = v;
        }
    } else {
        kvmax = scan(true);
    }
    K1P_SYNC();
    if (lane == 0 && nx.y > 0 && nx.z >= 0 && nx.x >= 0 && (int64_t)nx.x + nx.y + nx.z <= (int64_t)p.n_req) {
        const int64_t e0 = nx.x, e1 = e0 + nx.y + nx.z;
        prefetch_l2_bulk(p.req + e0, (uint32_t)(e1 - e0) * 16u);
        const int64_t d0 = e0 & ~1LL, d1 = min((e1 + 1) & ~1LL, (int64_t)p.n_req & ~1LL);   // 16-byte units
        if (d1 > d0) prefetch_l2_bulk(p.t_dead + d0, (uint32_t)(d1 - d0) * 8u);
    }
    int kvb = warp_max(kvmax);
    uint32_t st = kvb > in.kv_cap ? TP_ST_KV_OVER : 0u;

    // ---- FIFO gate (as k1_compact: one candidate at a time over its window, exact bound shortcut) ----
    int n_adm = allq ? nq : c0;
    const int ncand = allq ? 0 : forced >= 0 ? forced : nq;
    if (allq) {
        // the whole queue is in the histogram already
    } else if (forced < 0 && ncand > 0 && (st & TP_ST_KV_OVER)) {
        st |= TP_ST_QUEUE_BLOCKED;
    } else {
        int B1 = sv[0] >> 16;
        #pragma unroll 1
        for (int c = c0; c < ncand; ++c) {
            const int4 r = __ldg(&p.req[rb + nr + c]);
            const int q = r.y, lc = r.z;
            const int kvc_top = (int)fdN.div((uint32_t)(lc + q - 2)) + 1;
            if (forced < 0) {
                bool admit = B1 + 1 <= in.max_batch;
                if (admit && kvb + kvc_top > in.kv_cap) {
                    int mx = 0;
#pragma unroll 1
                    for (int m = 1 + lane; m <= lc; m += 32)
                        mx = max(mx, (sv[ph(m)] & 0xFFFF) + (int)fdN.div((uint32_t)(m + q - 2)) + 1);
                    mx = warp_max(mx);
                    admit = mx <= in.kv_cap;
                    kvb = max(kvb, mx);
                } else {
                    kvb += kvc_top;
                }
                if (!admit) {
                    st |= TP_ST_QUEUE_BLOCKED;
                    break;
                }
            } else {
                kvb += kvc_top;
            }
#pragma unroll 1
            for (int m = 1 + lane; m <= lc; m += 32) sv[ph(m)] += 65536 + (int)fdN.div((uint32_t)(m + q - 2)) + 1;
            K1P_SYNC();
            ++B1;
            ++n_adm;
            nloc = max(nloc, lc);
            lost |= (r.w & TP_REQ_LOST) || (c < 32 && ((lmask >> c) & 1u));
        }
    }
    if (forced >= 0 && forced < nq) st |= TP_ST_QUEUE_BLOCKED;
    const int n = nloc;
    if (n == 0) st |= TP_ST_EMPTY;
    else if (lost) st |= TP_ST_BYPASS_LOST;
    K1P_SYNC();

    if (p.B) {
        int* Bo = p.B + (int64_t)i * H;
        int* Ko = p.KV + (int64_t)i * H;
        const int lim = p.bkv_rows ? H : 1;
        #pragma unroll 1
        for (int m = 1 + lane; m <= lim; m += 32) {
            const int v = merged ? v1 : sv[ph(m)];    // merged: lim = 1, lane 0 holds m = 1
            Bo[m - 1] = v >> 16;
            Ko[m - 1] = v & 0xFFFF;
        }
    }
    if (lane == 0) {
        p.n[i] = n;
        p.n_adm[i] = n_adm;
        p.status[i] = st;
    }
    const int nn = (st & p.skip) ? 0 : n;
    const size_t row = (size_t)i * H;

    // ---- pieces (piece_rules) in lane segments: lane t walks m in [1 + t S2, 1 + (t+1) S2) ----
    // Pass A: the cell key (two rank-table lookups) and the head / end flags of each m, left in
    // place of the histogram word as key | head << 30 | fresh << 31 (keys < kMaxCells = 2^22);
    // a warp scan of the per-lane head counts gives every lane its first piece index; pass B writes
    // the piece records (first m, cell id), marks the fresh cells, and leaves in place of each m the
    // index of its piece -- which is what the Eq. 4 pass below looks up at every request's end.
    int h = 0, ends = 0;
    if (nn > 0) {
        const int n_sched = nr + n_adm;
#if TP_K1P_EQ4PF
        // the Eq. 4 pass's first record and deadline of this lane, in flight during the piece passes
        int2 qa = make_int2(0, 0);
        double qt = 0.0;
        if (lane < n_sched) {
            qa = make_int2(__ldg(&p.req[rb + lane].x), __ldg(&p.req[rb + lane].z));
            qt = __ldg(&p.t_dead[rb + lane]);
        }
#endif
        const uint32_t rtp = TP_K1P_RTP && (uint32_t)in.tp < 64u ? s_rtp[in.tp]
                                                     : rank_of(p.cuts + p.cut_off[0], p.cut_off[1] - p.cut_off[0], (float)in.tp);
        const uint32_t cell_base = rtp * (uint32_t)(p.cut_off[2] - p.cut_off[1] + 1) * nk1;
        const int S2 = s2_of(nn);
        const int mlo = 1 + lane * S2, mhi = min(mlo + S2 - 1, nn);     // empty when mlo > nn
        uint32_t pk = 0xffffffffu;                   // key / B of m - 1 (m = 1 always starts a piece)
        int pb = 0;
        if (!merged && mlo >= 2 && mlo <= nn) {
            const int v = sv[ph(mlo - 1)];
            pb = v >> 16;
            pk = key_of(v);
        }
        K1P_SYNC();                                   // every neighbour read before the in-place writes
        int32_t* const rec_m = p.run_m + row;
        uint32_t* const rec_k = p.run_key + row;
        long long* const D = p.end_d + row;
        int cnt = 0, e = 0;
        if (S2 <= 32) {
            // Mask form (n <= 1024): pass A leaves each iteration's cell key in place and sets bit
            // m - mlo of the lane's head mask; pass B visits only the set bits (one record per head,
            // not a pass per iteration), and the piece of an iteration l is base[t] + popc(mask[t]
            // up to l) - 1 (t the lane owning l), both left in the first 64 words for Eq. 4.
            uint32_t mask = mmask;                    // merged: pass A is done
            e = me;
            #pragma unroll 1
            for (int m0 = mlo; m0 <= (merged ? 0 : mhi); m0 += 4) {
                int4* const q = reinterpret_cast<int4*>(sv + ph(m0));
                int4 v = *q;
                const uint32_t bit = 1u << (m0 - mlo);
                auto flag = [&](int& x, uint32_t bu, bool live) {   // x: the histogram word of m
                    const uint32_t k = key_of(x);
                    const int b = x >> 16;
                    const bool endp = live && b < pb;         // m - 1 is an end position
                    const bool head = live && (k != pk || endp);
                    mask |= head ? bu : 0u;
                    e += endp;
                    x = (int)k;
                    pk = k;
                    pb = b;
                };
                flag(v.x, bit, true);
                flag(v.y, bit << 1, m0 + 1 <= mhi);
                flag(v.z, bit << 2, m0 + 2 <= mhi);
                flag(v.w, bit << 3, m0 + 3 <= mhi);
                *q = v;                                   // words past nn are never read again
            }
            cnt = __popc(mask);
            int x = cnt;                              // inclusive scan of the head counts
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(kFull, x, o);
                if (lane >= o) x += y;
            }
            h = __shfl_sync(kFull, x, 31);
            ends = __reduce_add_sync(kFull, e);
            const int base = x - cnt;                 // this lane's first piece
#if TP_K1P_BALB
            // balanced pass B: heads cluster at small m (most requests end early), so piece kk goes
            // to lane kk % 32 instead of the lane whose segment holds it; its owner t (the last lane
            // with base_t <= kk, by a shuffle binary search) and its bit (the (kk - base_t)-th set
            // bit of mask_t) give its m
            K1P_SYNC();                               // every lane's keys are in place
            #pragma unroll 1
            for (int k0 = 0; k0 < h; k0 += 32) {
                const int kk = k0 + lane;
                int t = 0;
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    const int bt = __shfl_sync(kFull, base, t + o);
                    if (bt <= kk) t += o;
                }
                const uint32_t mt = (uint32_t)__shfl_sync(kFull, (int)mask, t);
                const int jt = kk - __shfl_sync(kFull, base, t);
                if (kk < h) {
                    const int m = 1 + t * S2 + (int)__fns(mt, 0u, jt + 1);
                    const uint32_t k = cell_base + (uint32_t)sv[ph(m)];
                    *ptr_at(rec_m, (unsigned)kk) = m;
                    *ptr_at(rec_k, (unsigned)kk) = k;
                    claim_cell(p, k);                 // (also where a piece only repeats the cell)
                }
            }
#else
            int pos = base;
            #pragma unroll 1
            for (uint32_t mm = mask; mm; mm &= mm - 1, ++pos) {
                const int m = mlo + __ffs(mm) - 1;
                const uint32_t k = cell_base + (uint32_t)sv[ph(m)];
                *ptr_at(rec_m, (unsigned)pos) = m;
                *ptr_at(rec_k, (unsigned)pos) = k;
                claim_cell(p, k);                     // (also where a piece only repeats the cell)
            }
#endif
            #pragma unroll 1
            for (int k = lane; k < h; k += 32) D[k] = kNoDeadline;
            K1P_SYNC();                               // every lane's keys read
            sv[lane] = base;
            sv[32 + lane] = (int)mask;
            K1P_SYNC();                               // bases, masks and the initial minima in place
            // Eq. 4 per piece (piece_deadlines): end_d[k] = min over the scheduled requests whose
            // last iteration l is piece k's tail of ceil(fl64(t_dead - t_cur) * 2^40) (A-12), by a
            // fire-and-forget RED.MIN.S64 (a shared 64-bit atomicMin is a CAS loop)
            const uint32_t inv = ((1u << 20) + (uint32_t)S2 - 1) / (uint32_t)S2;   // (l-1)/S2, l-1 < 1024
#if TP_K1P_EQ4PF && TP_K1P_EQ4B > 1
            // batches of TP_K1P_EQ4B records per lane: the batch's loads are issued together (the
            // first one was loaded before the piece passes)
            #pragma unroll 1
            for (int j0 = lane; j0 < n_sched; j0 += 32 * TP_K1P_EQ4B) {
                int2 ab[TP_K1P_EQ4B];
                double tb[TP_K1P_EQ4B];
#pragma unroll
                for (int u = 0; u < TP_K1P_EQ4B; ++u) {
                    const int j = j0 + 32 * u;
                    ab[u] = make_int2(0, 1);
                    tb[u] = 0.0;
                    if (u == 0 && j0 == lane) {
                        ab[0] = qa;
                        tb[0] = qt;
                    } else if (j < n_sched) {
                        ab[u] = make_int2(__ldg(&p.req[rb + j].x), __ldg(&p.req[rb + j].z));
                        tb[u] = __ldg(&p.t_dead[rb + j]);
                    }
                }
#pragma unroll
                for (int u = 0; u < TP_K1P_EQ4B; ++u) {
                    if (j0 + 32 * u >= n_sched) break;
                    const int l1 = ab[u].y - ab[u].x - 1;   // 0 <= l - 1 < nn (validated; n = max l)
                    const long long d = slack_ticks(tb[u] - in.t_cur, p.tick_shift);
                    const int t = (int)(((uint32_t)l1 * inv) >> 20);
                    const int jj = l1 - t * S2;
                    const int k = sv[t] + __popc((uint32_t)sv[32 + t] & (0xffffffffu >> (31 - jj))) - 1;
                    if (d != kNoDeadline) atomicMin(ptr_at(D, (unsigned)k), d);
                }
            }
#else
            #pragma unroll 1
            for (int j = lane; j < n_sched; j += 32) {
#if TP_K1P_EQ4PF
                const int l1 = qa.y - qa.x - 1;       // 0 <= l - 1 < nn (validated; n = max l)
                const long long d = slack_ticks(qt - in.t_cur, p.tick_shift);
                if (j + 32 < n_sched) {
                    qa = make_int2(__ldg(&p.req[rb + j + 32].x), __ldg(&p.req[rb + j + 32].z));
                    qt = __ldg(&p.t_dead[rb + j + 32]);
                }
#else
                const int4 r = __ldg(&p.req[rb + j]);
                const int l1 = r.z - r.x - 1;         // 0 <= l - 1 < nn (validated; n = max l)
                const long long d = slack_ticks(__ldg(&p.t_dead[rb + j]) - in.t_cur, p.tick_shift);
#endif
                const int t = (int)(((uint32_t)l1 * inv) >> 20);
                const int jj = l1 - t * S2;
                const int k = sv[t] + __popc((uint32_t)sv[32 + t] & (0xffffffffu >> (31 - jj))) - 1;
                if (d != kNoDeadline) atomicMin(ptr_at(D, (unsigned)k), d);
            }
#endif
        } else {
            // Per-iteration form (long horizons): pass A leaves key | head << 30 | fresh << 31 in
            // place, pass B writes the records and leaves each iteration's piece index in place.
            #pragma unroll 1
            for (int m0 = mlo; m0 <= mhi; m0 += 4) {
                int4* const q = reinterpret_cast<int4*>(sv + ph(m0));
                int4 v = *q;
                const uint32_t k0 = key_of(v.x), k1 = key_of(v.y), k2 = key_of(v.z), k3 = key_of(v.w);
                auto flag = [&](int& x, uint32_t k, bool live) {
                    const int b = x >> 16;
                    const bool endp = live && b < pb;
                    const bool fresh = live && k != pk;
                    const bool head = fresh || endp;
                    cnt += head;
                    e += endp;
                    x = (int)(k | (head ? 1u << 30 : 0u) | (fresh ? 1u << 31 : 0u));
                    pk = k;
                    pb = b;
                };
                flag(v.x, k0, true);
                flag(v.y, k1, m0 + 1 <= mhi);
                flag(v.z, k2, m0 + 2 <= mhi);
                flag(v.w, k3, m0 + 3 <= mhi);
                *q = v;                               // words past nn are never read again
            }
            int x = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(kFull, x, o);
                if (lane >= o) x += y;
            }
            h = __shfl_sync(kFull, x, 31);
            ends = __reduce_add_sync(kFull, e);
            int pos = x - cnt;
            #pragma unroll 1
            for (int m0 = mlo; m0 <= mhi; m0 += 4) {
                int4* const q = reinterpret_cast<int4*>(sv + ph(m0));
                int4 v = *q;
                auto piece = [&](int& x, int m) {
                    const uint32_t w = (uint32_t)x;
                    if (w & (1u << 30)) {
                        const uint32_t k = cell_base + (w & 0x3fffffffu);
                        *ptr_at(rec_m, (unsigned)pos) = m;
                        *ptr_at(rec_k, (unsigned)pos) = k;
                        if (w >> 31) claim_cell(p, k);
                        ++pos;
                    }
                    x = pos - 1;
                };
                piece(v.x, m0);
                piece(v.y, m0 + 1);
                piece(v.z, m0 + 2);
                piece(v.w, m0 + 3);
                *q = v;
            }
            #pragma unroll 1
            for (int k = lane; k < h; k += 32) D[k] = kNoDeadline;
            K1P_SYNC();
            #pragma unroll 1
            for (int j = lane; j < n_sched; j += 32) {
                const int4 r = __ldg(&p.req[rb + j]);
                const int l = r.z - r.x;
                const long long d = slack_ticks(__ldg(&p.t_dead[rb + j]) - in.t_cur, p.tick_shift);
                if (d != kNoDeadline) atomicMin(ptr_at(D, (unsigned)sv[ph(l)]), d);
            }
        }
    }
    if (lane == 0) {
        p.run_h[i] = h;
        p.end_n[i] = nn > 0 ? ends + 1 : 0;           // + m = nn, always an end
    }
#if TP_K1P_ZDIRTY
    // words this instance can have written: events at <= n + 1, in-place keys / piece indices of
    // 4-iteration batches at <= n + 3, bases and masks in the first 64; everything past them is
    // still 0 (the scanned words past n + 1 are 0), so the next instance clears only this prefix
    zhi = min(p.arr, max(64, (ph(min(n + 4, H + 1)) + 4) & ~3));
#endif
    }
}

template <int WPI, bool FLAGGED = false>   // FLAGGED: the instances k1_packed handed over
__global__ void __launch_bounds__(cta_warps<WPI>() * 32, WPI == 1 ? 6 : 32 / cta_warps<WPI>())
k1_compact(const __grid_constant__ K1cParams p) {
    extern __shared__ __align__(16) int smem[];
    constexpr int NG = cta_warps<WPI>() / WPI;         // groups (instances) per full CTA
    __shared__ long long s_x[WPI > 1 ? NG : 1][2 * WPI * 4];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g = w / WPI, gpb = (int)(blockDim.x >> 5) / WPI;
    Group<WPI> grp;
    grp.gw = w % WPI;
    grp.bar = 1 + g;
    grp.xs = s_x[WPI > 1 ? g : 0];
    const int gl = grp.gw * 32 + lane;                 // lane within the group
    int* sB = smem + (size_t)g * 2 * p.arr;
    int* sKV = sB + p.arr;
    if constexpr (FLAGGED) {  // persistent over the hand-over list
        const int nflag = *p.flag_count + 1;
        for (int j = blockIdx.x * gpb + g; j < nflag; j += gridDim.x * gpb) {
            grp.sync();
            k1_body<WPI>(p, p.flag_list[j], grp, sB, sKV, gl, lane);
        }
        return;
    }
    const int i = blockIdx.x * gpb + g;
    if (i >= p.n_inst) return;                         // group-uniform
    k1_body<WPI>(p, i, grp, sB, sKV, gl, lane);
}

// After K1c: every cell marked seen (claim_cell) gets the next index of the cell list K2 evaluates
// (cell_count holds count - 1; the order of the list is immaterial: K2 and K3c address the LUT by
// cell id) and a zero clamp mask.  Cells listed by an earlier launch on the same workspace keep
// their index.
__global__ void __launch_bounds__(256) k1_cells_collect(int32_t* cell_tab, int32_t n_cells, uint32_t* cell_list,
                                                        int32_t* cell_count, uint32_t* cell_clamp) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x, lane = threadIdx.x & 31;
    const bool seen = k < n_cells && cell_tab[k] == kCellSeen;
    const unsigned b = __ballot_sync(kFull, seen);
    if (!b) return;                                    // warp-uniform
    int base = 0;
    if (lane == 0) base = atomicAdd(cell_count, __popc(b)) + 1;
    base = __shfl_sync(kFull, base, 0);
    if (seen) {
        const int idx = base + __popc(b & ((1u << lane) - 1u));
        cell_list[idx] = (uint32_t)k;
        cell_tab[k] = idx;
        cell_clamp[k] = 0u;
    }
}

}  // namespace

int project_compact_smem_per_warp(int32_t H) { return 2 * seg_geom(H, 32).arr * (int)sizeof(int); }

namespace {
int env_int_k1(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

// TP_K1C_WARPS (1/2/4): warps per instance override (tuning)
int env_wpi() {
    const char* v = std::getenv("TP_K1C_WARPS");
    const int x = v ? std::atoi(v) : 0;
    return (x == 1 || x == 2 || x == 4 || x == 8) ? x : 0;
}

template <int WPI, bool FLAGGED = false>
int launch_wpi(const K1cParams& p0, int32_t n_inst, int32_t H, cudaStream_t s) {
    K1cParams p = p0;
    const SegGeom g = seg_geom(H, 32 * WPI);
    p.S_log2 = g.S_log2;
    p.P = g.P;
    p.arr = g.arr;
    // instances per CTA: up to kWarpsPerCta / WPI, fewer for long horizons (per-group histograms)
    const size_t per_group = (size_t)2 * g.arr * sizeof(int);
    if (per_group > 200 * 1024) return TP_EINVAL;
    const int gpb = (int)std::max<size_t>(1, std::min<size_t>(cta_warps<WPI>() / WPI, (100 * 1024) / per_group));
    const size_t smem = (size_t)gpb * per_group;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return TP_ECUDA;
    static int attr_bytes[64] = {};
    if (dev < 64 && attr_bytes[dev] < (int)smem) {
        if (cudaFuncSetAttribute(k1_compact<WPI, FLAGGED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess)
            return TP_EINVAL;   // H too large for the per-group histograms
        attr_bytes[dev] = (int)smem;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // FLAGGED: a persistent grid over the (normally empty) hand-over list
    const int grid = FLAGGED ? std::min(sms, (n_inst + gpb - 1) / gpb) : (n_inst + gpb - 1) / gpb;
    k1_compact<WPI, FLAGGED><<<grid, gpb * WPI * 32, smem, s>>>(p);
    return cudaPeekAtLastError() == cudaSuccess ? TP_OK : TP_ECUDA;
}

// k1_packed (one warp per instance), then the wide kernel over the instances it handed over
int launch_packed(const K1cParams& p0, int32_t n_inst, int32_t H, cudaStream_t s) {
    K1cParams p = p0;
    const SegGeom g = seg_geom(H, 32);
    p.S_log2 = g.S_log2;
    p.P = g.P;
    int arr = g.arr;
#if TP_K1P_LINEAR
    {   // unpadded: the S2-segment passes touch words < 32 S2(H) (S2 is monotone in n), the events
        // and the cleared prefix words <= H + 4
        int S2 = (((H + 31) >> 5) + 3) & ~3;
        if ((S2 & 4) == 0 && 32 * (S2 - 4) < H && S2 + 4 <= 32) S2 += 4;
        arr = (std::max(32 * S2, H + 8) + 3) & ~3;
    }
#endif
    p.arr = arr;
    const size_t per_warp = (size_t)arr * sizeof(int);
    if (per_warp > 200 * 1024) return TP_EINVAL;
    // rank tables in shared memory when they are small next to the histograms (the model's cut sets)
    const int tab_entries = p.rtab_off[1] + p.rtab_len[1];
    const size_t tab_bytes = ((size_t)tab_entries * 2 + 15) & ~(size_t)15;
    constexpr size_t kCtaSmem = 75 * 1024;            // three CTAs per SM
    const bool st = TP_K1P_ST && tab_bytes <= 32 * 1024 && tab_bytes + per_warp <= kCtaSmem;
    p.tab_words = st ? (int32_t)(tab_bytes / 4) : 0;
    const size_t room = st ? kCtaSmem - tab_bytes : (size_t)100 * 1024;
    const int wpb = (int)std::max<size_t>(1, std::min<size_t>(TP_K1P_WARPS, room / per_warp));
    const size_t smem = (st ? tab_bytes : 0) + (size_t)wpb * per_warp;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return TP_ECUDA;
    auto go = [&](auto kern, int li) {
        static int attr_bytes[2][64] = {}, occ_smem[2][64] = {}, occ_blocks[2][64] = {}, occ_wpb[2][64] = {};
        if (dev < 64 && attr_bytes[li][dev] < (int)smem) {
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return TP_EINVAL;
            attr_bytes[li][dev] = (int)smem;
        }
        // persistent: as many CTAs as fit at once
        if (dev < 64 && (occ_smem[li][dev] != (int)smem || occ_wpb[li][dev] != wpb)) {
            int b = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, wpb * 32, smem);
            occ_blocks[li][dev] = b > 0 ? b : 1;
            occ_smem[li][dev] = (int)smem;
            occ_wpb[li][dev] = wpb;
        }
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int grid = (int)std::min<int64_t>((n_inst + wpb - 1) / wpb, (int64_t)sms * (dev < 64 ? occ_blocks[li][dev] : 1));
        kern<<<grid, wpb * 32, smem, s>>>(p);
        return cudaPeekAtLastError() == cudaSuccess ? TP_OK : TP_ECUDA;
    };
    const int rc = st ? go(k1_packed<true>, 1) : go(k1_packed<false>, 0);
    if (rc != TP_OK) return rc;
    return launch_wpi<1, true>(p0, n_inst, H, s);
}
}  // namespace

int launch_project_compact(const K2Params& w, const tp_inst* inst, int32_t n_inst, const tp_req* req,
                           int32_t n_req, const double* t_dead, int32_t H, int32_t* B, int32_t* KV, int bkv_rows,
                           int32_t* n, int32_t* n_adm, uint32_t* status, uint32_t skip, cudaStream_t s,
                           const int32_t* force_adm, const uint32_t* lost_mask) {
    if (n_inst == 0) return TP_OK;
    if (!w.cell_tab || !w.end_n || !w.k1_next) return TP_EINVAL;
    K1cParams p;
    p.inst = inst;
    p.req = reinterpret_cast<const int4*>(req);
    p.t_dead = t_dead;
    p.n_inst = n_inst;
    p.n_req = n_req;
    p.H = H;
    p.B = B;
    p.KV = KV;
    p.bkv_rows = bkv_rows;
    p.n = n;
    p.n_adm = n_adm;
    p.status = status;
    p.force_adm = force_adm;
    p.lost_mask = lost_mask;
    p.skip = skip;
    p.cuts = w.cuts;
    for (int k = 0; k < 5; ++k) p.cut_off[k] = w.cut_off[k];
    p.rtab = w.rtab;
    for (int k = 0; k < 2; ++k) {
        p.rtab_off[k] = w.rtab_off[k];
        p.rtab_len[k] = w.rtab_len[k];
    }
    p.run_h = w.run_h;
    p.run_m = w.run_m;
    p.run_key = w.run_key;
    p.cell_tab = w.cell_tab;
    p.cell_list = w.cell_list;
    p.cell_count = w.cell_count;
    p.cell_clamp = w.cell_clamp;
    p.end_n = w.end_n;
    p.end_d = w.end_d;
    p.tick_shift = w.tick_shift;
    p.next = w.k1_next;
    p.flag_count = w.flag_count;
    p.flag_list = w.flag_list;
    // K3c's counters, flag_count, cell_count (all count - 1) and cell_tab are contiguous: one reset; claimers zero
    // their cells' clamp masks
    if (cudaMemsetAsync(w.k1_next, 0xFF, 20 + (size_t)w.n_cells * 4, s) != cudaSuccess) return TP_ECUDA;
    // warps per instance: small batches get several warps per instance (the per-instance chain
    // of dependent loads and reductions is the latency; shorter per-warp loops shorten it), large
    // batches one (the GPU is full anyway)
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static const int wpi_env = env_wpi();
    const int64_t slots = (int64_t)sms * 32;    // C2 (1,024 instances): 4 warps each; C3: one
    const int wpi = wpi_env ? wpi_env : ((int64_t)n_inst * 4 <= slots ? 4 : (int64_t)n_inst * 2 <= slots ? 2 : 1);
    static const bool packed = env_int_k1("TP_K1C_PACKED", 1) != 0;
    int rc;
    switch (wpi) {
        case 8: rc = launch_wpi<8>(p, n_inst, H, s); break;
        case 4: rc = launch_wpi<4>(p, n_inst, H, s); break;
        case 2: rc = launch_wpi<2>(p, n_inst, H, s); break;
        default: rc = packed ? launch_packed(p, n_inst, H, s) : launch_wpi<1>(p, n_inst, H, s); break;
    }
    if (rc != TP_OK) return rc;
    constexpr int kCollectThreads = 256;
    k1_cells_collect<<<(w.n_cells + kCollectThreads - 1) / kCollectThreads, kCollectThreads, 0, s>>>(
        w.cell_tab, w.n_cells, w.cell_list, w.cell_count, w.cell_clamp);
    return cudaPeekAtLastError() == cudaSuccess ? TP_OK : TP_ECUDA;
}

}  // namespace tp
