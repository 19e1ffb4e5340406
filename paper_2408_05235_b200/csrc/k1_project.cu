// K1 -- KV usage & batch-size projection (PAPER §4.2, Eq. 1-2) with the FIFO
// admission gate (check 1 + batch cap, §4.3.2, one request at a time P:755).
//
// One CTA per instance.  Instead of evaluating Eq. 1 for every (request, m) pair, every request
// contributes O(l/N) integer events to two difference arrays in shared memory:
//   B : +1 at m = 1, -1 at m = l + 1
//   KV: +ceil((a + q) / N) at m = 1, +1 at every m in [2, l] where the request's token count
//       a + q + m - 1 crosses a block boundary ((a + q + m - 2) % N == 0), and -ceil((a+q+l-1)/N)
//       at m = l + 1
// and a block-wide inclusive scan turns them into B[m], KV[m] (equal to Eq. 1-2 exactly; pinned by
// tests/test_gpu_parity.py against the oracle's direct Eq. 1 sums).  HBM traffic: 16 B per request
// read + 8 B per (instance, m <= H) written.
#include "tp_internal.cuh"

namespace tp {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kGate = 8;        // queued candidates evaluated per block reduction

// Scan segment per thread: a multiple of 4 iterations (128-bit shared loads), and the padded array
// length so that every segment [1 + t*S, 1 + (t+1)*S) lies inside it.
__host__ __device__ __forceinline__ int seg_len(int H) { return ((H + 4 * kThreads - 1) / (4 * kThreads)) * 4; }
__host__ __device__ __forceinline__ int seg_pad(int H) { return ((H + 1 + 3) / 4) * 4 + 4; }

__device__ __forceinline__ int64_t block_sum64(int64_t v, int64_t* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) s += red[i];
    return s;
}

__device__ __forceinline__ int block_max(int v, int* red) {
    v = __reduce_max_sync(0xffffffffu, v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    int s = red[0];
#pragma unroll
    for (int i = 1; i < kWarps; ++i) s = max(s, red[i]);
    return s;
}

__global__ void __launch_bounds__(kThreads, 4)
k1_project(const tp_inst* __restrict__ inst, const int4* __restrict__ req, int32_t n_req, int32_t H,
           int32_t* __restrict__ Bout, int32_t* __restrict__ KVout, int32_t* __restrict__ nout,
           int32_t* __restrict__ nadm_out, uint32_t* __restrict__ status, const int32_t* __restrict__ force_adm,
           const uint32_t* __restrict__ lost_mask) {
    extern __shared__ __align__(16) int smem[];
    // index m in [1, Hp]; &sB[1] and &sKV[1] 16-byte aligned so a thread's 4-aligned segment of m
    // is read with 128-bit loads (conflict-free)
    const int Hp = seg_pad(H);
    int* sB = smem + 3;
    int* sKV = smem + 3 + Hp;
    __shared__ int64_t red64[kWarps];
    __shared__ int redi[kWarps];
    __shared__ int s_admit;
    __shared__ int s_gate[kWarps][kGate];

    const int i = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const tp_inst in = inst[i];
    const int64_t rb = in.req_begin;
    const int nr = in.n_run, nq = in.n_queue, N = in.N;
    // the divider for N is a per-instance constant: one thread builds it (64-bit division)
    __shared__ FastDiv s_fd;
    if (tid == 0) s_fd = FastDiv((uint32_t)(N > 0 ? N : 1));

    for (int m = tid; m < Hp; m += kThreads) sB[m] = sKV[m] = 0;

    // ---- validation (include/tp.h conventions) ----
    bool bad = N < 1 || in.tp < 1 || (int64_t)in.tp >= kFeatLimit || nr < 0 || nq < 0 || in.kv_cap < 0 ||
               in.max_batch < 0 || rb < 0 || rb + (int64_t)nr + nq > (int64_t)n_req;
    int64_t foot = 0;
    __syncthreads();
    const FastDiv fdN = s_fd;
    if (!bad) {
        for (int e = tid; e < nr + nq; e += kThreads) {
            const int4 r = __ldg(&req[rb + e]);
            const int64_t l = (int64_t)r.z - r.x;
            const bool eb = r.x < 0 || r.y < 1 || r.z < 1 || r.x >= kFeatLimit || r.y >= kFeatLimit || l < 1 ||
                            l > H || (e >= nr && r.x != 0);
            bad |= eb;
            if (!eb) foot += (int64_t)fdN.div((uint32_t)(r.x + l - 2 + r.y)) + 1;   // ceil((a+l-1+q)/N)
        }
    }
    bad = __syncthreads_or(bad);   // (also publishes s_fd)
    if (!bad) bad = block_sum64(foot, red64) >= kFeatLimit;
    if (bad) {
        for (int m = tid; m < H; m += kThreads) {
            Bout[(int64_t)i * H + m] = 0;
            KVout[(int64_t)i * H + m] = 0;
        }
        if (tid == 0) {
            nout[i] = 0;
            nadm_out[i] = 0;
            status[i] = TP_ST_BAD_INPUT;
        }
        return;
    }

    // ---- running requests -> event histograms (Eq. 1 increments) ----
    int nloc = 0, b1 = 0, kv1 = 0;
    bool lost = false;
    for (int e = tid; e < nr; e += kThreads) {
        const int4 r = __ldg(&req[rb + e]);
        const int a = r.x, q = r.y, l = r.z - r.x;
        nloc = max(nloc, l);
        lost |= (r.w & TP_REQ_LOST) != 0;
        const int aq = a + q;
        atomicAdd(&sB[l + 1], -1);
        const int c1 = (int)fdN.div((uint32_t)(aq - 1));                 // ceil(aq / N) - 1, aq >= 1
        kv1 += c1 + 1;
        ++b1;
        // first m >= 2 with (aq + m - 2) % N == 0, then every N iterations (m <= l <= H: no overflow)
        for (int m = 2 + (c1 + 1) * N - aq; m <= l; m += N) atomicAdd(&sKV[m], 1);
        atomicAdd(&sKV[l + 1], -((int)fdN.div((uint32_t)(aq + l - 2)) + 1));   // -ceil((aq + l - 1) / N)
    }
    // the m = 1 terms of every request: one shared atomic per warp
    b1 = __reduce_add_sync(0xffffffffu, b1);
    kv1 = __reduce_add_sync(0xffffffffu, kv1);
    if (lane == 0 && b1) {
        atomicAdd(&sB[1], b1);
        atomicAdd(&sKV[1], kv1);
    }
    lost = __syncthreads_or(lost);

    // ---- inclusive scans: thread t owns the contiguous segment [lo, hi) of m ----
    const int S = seg_len(H);
    int kvmax = 0;
    const int lo = 1 + tid * S, hi = min(lo + S, H + 1);
    {
        int sb = 0, skv = 0;
        for (int m = lo; m < hi; m += 4) {     // 4-aligned segment, zero padding past H
            const int4 b = *reinterpret_cast<const int4*>(sB + m);
            const int4 k = *reinterpret_cast<const int4*>(sKV + m);
            sb += b.x + b.y + b.z + b.w;
            skv += k.x + k.y + k.z + k.w;
        }
        // exclusive block scan of the (sb, skv) pairs
        int xb = sb, xkv = skv;
        const int w = warp;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int yb = __shfl_up_sync(0xffffffffu, xb, o), ykv = __shfl_up_sync(0xffffffffu, xkv, o);
            if (lane >= o) {
                xb += yb;
                xkv += ykv;
            }
        }
        __shared__ int wb[kWarps], wkv[kWarps];
        if (lane == 31) {
            wb[w] = xb;
            wkv[w] = xkv;
        }
        __syncthreads();
        int pb = xb - sb, pkv = xkv - skv;
        for (int k = 0; k < w; ++k) {
            pb += wb[k];
            pkv += wkv[k];
        }
        for (int m = lo; m < hi; m += 4) {
            int4 b = *reinterpret_cast<const int4*>(sB + m);
            int4 k = *reinterpret_cast<const int4*>(sKV + m);
            b.x += pb; b.y += b.x; b.z += b.y; b.w += b.z;
            k.x += pkv; k.y += k.x; k.z += k.y; k.w += k.z;
            pb = b.w;
            pkv = k.w;
            *reinterpret_cast<int4*>(sB + m) = b;
            *reinterpret_cast<int4*>(sKV + m) = k;
            // positions past H are padding (their events are zero; never read as outputs)
            kvmax = max(kvmax, max(max(k.x, m + 1 <= H ? k.y : 0), max(m + 2 <= H ? k.z : 0, m + 3 <= H ? k.w : 0)));
        }
    }
    __syncthreads();

    uint32_t st = block_max(kvmax, redi) > in.kv_cap ? TP_ST_KV_OVER : 0u;

    // ---- FIFO gate: queued c admitted iff B[1]+1 <= max_batch and max_m KV + KV_c <= kv_cap ----
    // Candidates are taken in batches of kGate: admitting c means admitting the whole prefix before
    // it, so one pass computes, for every prefix p of the batch, max_m (KV[m] + sum_{j<=p} KV_j[m]);
    // the first prefix over the cap (or over max_batch) stops the queue.  Same result as one
    // candidate at a time, with one block reduction per batch instead of per candidate.
    int n_adm = 0;
    bool blocked = false;
    // forced mode (admission control, tp_decide_admit): admit exactly force_adm[i] candidates (the
    // SLO checks were made at f_max beforehand), with lost_mask[i] marking the "lost" ones
    const int forced = force_adm ? min(max(force_adm[i], 0), nq) : -1;
    const uint32_t lmask = lost_mask ? lost_mask[i] : 0u;
    for (int c0 = 0; c0 < (forced >= 0 ? forced : nq) && !blocked; c0 += kGate) {
        const int cn = min(kGate, (forced >= 0 ? forced : nq) - c0);
        int q[kGate], lc[kGate], mx[kGate];
        uint32_t lostmask = 0;
#pragma unroll
        for (int j = 0; j < kGate; ++j) {
            q[j] = 1;
            lc[j] = 0;
            mx[j] = 0;
            if (j < cn) {
                const int4 r = __ldg(&req[rb + nr + c0 + j]);
                q[j] = r.y;
                lc[j] = r.z;
                if ((r.w & TP_REQ_LOST) || (c0 + j < 32 && ((lmask >> (c0 + j)) & 1u))) lostmask |= 1u << j;
            }
        }
        // candidate j's Eq. 1 blocks over this thread's segment, incrementally: kv = ceil(t / N) with
        // t = m - 1 + q tokens and d = (t - 1) mod N; m -> m + 1 adds a block when d wraps to 0
        int kvj[kGate], dj[kGate];
#pragma unroll
        for (int j = 0; j < kGate; ++j) {
            kvj[j] = dj[j] = 0;
            if (j < cn) {
                const int t1 = lo + q[j] - 2;          // t - 1 at m = lo (>= 0)
                kvj[j] = (int)fdN.div((uint32_t)t1) + 1;
                dj[j] = t1 - (kvj[j] - 1) * N;
            }
        }
        int maxlc = 0;
#pragma unroll
        for (int j = 0; j < kGate; ++j) maxlc = max(maxlc, lc[j]);
        const int mlim = min(hi, maxlc + 1);     // past every candidate's window only KV[m] counts
        for (int m4 = lo; m4 < mlim; m4 += 4) {
            const int4 kv4 = *reinterpret_cast<const int4*>(sKV + m4);
            const int kvs[4] = {kv4.x, kv4.y, kv4.z, kv4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int m = m4 + u;
                if (m < mlim) {
                    int run = kvs[u];
#pragma unroll
                    for (int j = 0; j < kGate; ++j) {
                        if (j < cn) {
                            run += (m <= lc[j]) ? kvj[j] : 0;
                            if (++dj[j] == N) {
                                dj[j] = 0;
                                ++kvj[j];
                            }
                        }
                        mx[j] = max(mx[j], run);
                    }
                }
            }
        }
        int tail = 0;
        for (int m = max(lo, mlim); m < hi; ++m) tail = max(tail, sKV[m]);
#pragma unroll
        for (int j = 0; j < kGate; ++j) mx[j] = max(mx[j], tail);
#pragma unroll
        for (int j = 0; j < kGate; ++j) mx[j] = __reduce_max_sync(0xffffffffu, mx[j]);
        if (lane == 0)
#pragma unroll
            for (int j = 0; j < kGate; ++j) s_gate[warp][j] = mx[j];
        __syncthreads();
        if (tid == 0 && forced >= 0) {
            s_admit = cn;
        } else if (tid == 0) {
            int p = 0;
            while (p < cn) {
                int M = 0;
                for (int w = 0; w < kWarps; ++w) M = max(M, s_gate[w][p]);
                if (sB[1] + p + 1 > in.max_batch || M > in.kv_cap) break;
                ++p;
            }
            s_admit = p;
        }
        __syncthreads();
        const int p = s_admit;
        if (p > 0) {
#pragma unroll
            for (int j = 0; j < kGate; ++j)
                if (j < p) {
                    const int t1 = lo + q[j] - 2;
                    kvj[j] = (int)fdN.div((uint32_t)t1) + 1;
                    dj[j] = t1 - (kvj[j] - 1) * N;
                }
            for (int m4 = lo; m4 < mlim; m4 += 4) {
                int add[4] = {0, 0, 0, 0}, addb[4] = {0, 0, 0, 0};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int m = m4 + u;
                    if (m < mlim) {
#pragma unroll
                        for (int j = 0; j < kGate; ++j)
                            if (j < p) {
                                if (m <= lc[j]) {
                                    add[u] += kvj[j];
                                    ++addb[u];
                                }
                                if (++dj[j] == N) {
                                    dj[j] = 0;
                                    ++kvj[j];
                                }
                            }
                    }
                }
                int4 k = *reinterpret_cast<int4*>(sKV + m4);
                int4 b = *reinterpret_cast<int4*>(sB + m4);
                k.x += add[0]; k.y += add[1]; k.z += add[2]; k.w += add[3];
                b.x += addb[0]; b.y += addb[1]; b.z += addb[2]; b.w += addb[3];
                *reinterpret_cast<int4*>(sKV + m4) = k;
                *reinterpret_cast<int4*>(sB + m4) = b;
            }
        }
#pragma unroll
        for (int j = 0; j < kGate; ++j)
            if (j < p) {
                nloc = max(nloc, lc[j]);
                lost |= (lostmask >> j) & 1u;
            }
        n_adm += p;
        if (p < cn) {
            blocked = true;
            st |= TP_ST_QUEUE_BLOCKED;
        }
        __syncthreads();
    }
    if (forced >= 0 && forced < nq) st |= TP_ST_QUEUE_BLOCKED;
    const int n = block_max(nloc, redi);

    if ((H & 3) == 0) {   // rows 16-byte aligned: 128-bit stores
        int4* b4 = reinterpret_cast<int4*>(Bout + (int64_t)i * H);
        int4* k4 = reinterpret_cast<int4*>(KVout + (int64_t)i * H);
        for (int v = tid; v < (H >> 2); v += kThreads) {
            const int m = 4 * v + 1;
            b4[v] = *reinterpret_cast<const int4*>(sB + m);
            k4[v] = *reinterpret_cast<const int4*>(sKV + m);
        }
    } else {
        for (int m = tid; m < H; m += kThreads) {
            Bout[(int64_t)i * H + m] = sB[m + 1];
            KVout[(int64_t)i * H + m] = sKV[m + 1];
        }
    }
    if (tid == 0) {
        if (n == 0) st |= TP_ST_EMPTY;
        else if (lost) st |= TP_ST_BYPASS_LOST;
        nout[i] = n;
        nadm_out[i] = n_adm;
        status[i] = st;
    }
}

}  // namespace

int launch_project(const tp_inst* inst, int32_t n_inst, const tp_req* req, int32_t n_req, int32_t H,
                   int32_t* B, int32_t* KV, int32_t* n, int32_t* n_adm, uint32_t* status, cudaStream_t s,
                   const int32_t* force_adm, const uint32_t* lost_mask) {
    if (n_inst == 0) return TP_OK;
    const size_t smem = (size_t)(4 + 2 * seg_pad(H)) * sizeof(int);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return TP_ECUDA;
    static bool attr_done[64] = {};
    if (dev < 64 && !attr_done[dev]) {
        if (cudaFuncSetAttribute(k1_project, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (4 + 2 * seg_pad(kMaxH)) * (int)sizeof(int)) != cudaSuccess)
            return TP_ECUDA;
        attr_done[dev] = true;
    }
    k1_project<<<n_inst, kThreads, smem, s>>>(inst, reinterpret_cast<const int4*>(req), n_req, H, B, KV, n,
                                                n_adm, status, force_adm, lost_mask);
    return cudaPeekAtLastError() == cudaSuccess ? TP_OK : TP_ECUDA;
}

}  // namespace tp
