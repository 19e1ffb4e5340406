// Full admission control on the GPU (PAPER §4.3.2): every queued request,
// in FIFO order, must pass check 1 (KV capacity, + batch cap), check 2 (mean TBT at the maximum
// frequency) and check 3 (Eq. 4 for every scheduled request at the maximum frequency) on the state
// with it virtually appended; if only its own deadline fails it is scheduled but marked "lost".
//
// The candidates of one instance are decided one at a time, but the state that decides candidate p
// is always "running + the first p queued" (the admitted set is a FIFO prefix), so every prefix is
// evaluated in parallel as a virtual instance, and a sequential scan over the per-prefix results
// resolves the admitted count and the lost marks:
//   k_admit_expand   virtual instance (i, p) = instance i with its first p queued requests forced in,
//                    for p <= the check-1 prefix (K1's gate) and p <= q_max
//   [K1 forced, K2 cell mode at F = 1 (f_max) on the virtual instances]
//   k_admit_checks   per virtual instance: T_R at f_max per run (exact ticks), TBT, and the Eq. 4
//                    outcome of every scheduled request (bit per candidate, one flag for the running)
//   k_admit_resolve  per instance: scan p = 1.. (admit / admit as lost / stop)
#include "tp_internal.cuh"

namespace tp {
namespace {

constexpr int kThreads = 128;

__global__ void k_admit_expand(const tp_inst* __restrict__ inst, int32_t n_inst, int32_t qc,
                               const int32_t* __restrict__ n_adm1, const uint32_t* __restrict__ status1,
                               tp_inst* __restrict__ vinst, int32_t* __restrict__ vforce) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= (int64_t)n_inst * qc) return;
    const int i = (int)(v / qc), p = (int)(v % qc) + 1;
    tp_inst in = inst[i];
    const bool active = !(status1[i] & TP_ST_BAD_INPUT) && p <= n_adm1[i];
    if (!active) in.N = 0;            // -> BAD_INPUT: skipped by every later kernel
    else in.n_queue = p;
    vinst[v] = in;
    vforce[v] = active ? p : 0;
}

struct CheckParams {
    const tp_inst* vinst;
    const int4* req;
    const double* t_dead;
    const int32_t* vn;
    const uint32_t* vstatus;
    const int32_t* run_h;
    const int32_t* run_m;
    const uint32_t* run_key;
    const int32_t* cell_tab;
    const float* lut;
    int32_t H;
    long long tbt_ticks;
    uint2* vres;   // x = candidate fail mask, y = flags (1 valid, 2 TBT ok, 4 a running request fails)
};

__global__ void __launch_bounds__(kThreads)
k_admit_checks(const __grid_constant__ CheckParams p) {
    extern __shared__ long long sm[];   // r_before[h] | r_t[h] | r_start[h + 1] (int)
    __shared__ long long s_carry;
    const int v = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (p.vstatus[v] & TP_ST_BAD_INPUT) {
        if (tid == 0) p.vres[v] = make_uint2(0u, 0u);
        return;
    }
    const tp_inst in = p.vinst[v];
    const int n = p.vn[v];
    const size_t row = (size_t)v * p.H;
    const int h = p.run_h[v];
    long long* r_before = sm;
    long long* r_t = sm + h;
    int* r_start = reinterpret_cast<int*>(sm + 2 * h);
    if (tid == 0) s_carry = 0;
    for (int k = tid; k < h; k += kThreads) r_start[k] = p.run_m[row + k];
    if (tid == 0) r_start[h] = n + 1;
    __syncthreads();
    // T_R before each run at f_max: block-wide exclusive scan of len_k * t_k (exact int64 ticks)
    for (int k0 = 0; k0 < h; k0 += kThreads) {
        const int k = k0 + tid;
        long long t = 0, own = 0;
        if (k < h) {
            const float ips = __ldg(p.lut + __ldg(p.cell_tab + p.run_key[row + k]));   // F = 1: the f_max row
            t = (long long)(__frcp_rn(ips) * 0x1p40f);
            own = (long long)(r_start[k + 1] - r_start[k]) * t;
        }
        long long x = own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        __shared__ long long wsum[kThreads / 32];
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        long long before = s_carry;
        for (int w = 0; w < warp; ++w) before += wsum[w];
        if (k < h) {
            r_before[k] = before + x - own;
            r_t[k] = t;
        }
        __syncthreads();
        if (tid == 0)
            for (int w = 0; w < kThreads / 32; ++w) s_carry += wsum[w];
        __syncthreads();
    }
    const long long total = s_carry;   // T_R[n]
    // Eq. 4 for every scheduled request (running + the p forced candidates), lost ones ignored
    const int n_sched = in.n_run + in.n_queue;
    uint32_t mask = 0;
    bool run_fail = false;
    for (int e = tid; e < n_sched; e += kThreads) {
        const int64_t j = (int64_t)in.req_begin + e;
        const int4 r = __ldg(&p.req[j]);
        if (r.w & TP_REQ_LOST) continue;
        const int l = r.z - r.x;
        int lo = 0, hi = h;   // last run with start <= l
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (r_start[mid] <= l) lo = mid;
            else hi = mid;
        }
        const long long TR = r_before[lo] + (long long)(l - r_start[lo] + 1) * r_t[lo];
        const bool fail = !(TR < slack_ticks(__ldg(&p.t_dead[j]) - in.t_cur));
        if (fail) {
            if (e < in.n_run) run_fail = true;
            else mask |= 1u << (e - in.n_run);
        }
    }
    for (int o = 16; o; o >>= 1) mask |= __shfl_xor_sync(0xffffffffu, mask, o);
    run_fail = __syncthreads_or(run_fail);
    __shared__ uint32_t smask;
    if (tid == 0) smask = 0;
    __syncthreads();
    if (lane == 0 && mask) atomicOr(&smask, mask);
    __syncthreads();
    if (tid == 0) {
        const bool tbt_ok = total <= (long long)n * p.tbt_ticks;   // check 2
        p.vres[v] = make_uint2(smask, 1u | (tbt_ok ? 2u : 0u) | (run_fail ? 4u : 0u));
    }
}

__global__ void k_admit_resolve(int32_t n_inst, int32_t qc, const tp_inst* __restrict__ inst,
                                const uint32_t* __restrict__ status1, const int32_t* __restrict__ n_adm1,
                                const uint2* __restrict__ vres, int32_t* __restrict__ n_adm,
                                uint32_t* __restrict__ lost) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_inst) return;
    int adm = 0;
    uint32_t marked = 0;
    if (!(status1[i] & TP_ST_BAD_INPUT)) {
        const int pmax = min(n_adm1[i], qc);
        for (int pp = 1; pp <= pmax; ++pp) {
            const uint2 r = vres[(int64_t)i * qc + pp - 1];
            if (!(r.y & 1u)) break;
            const uint32_t prior = r.x & ((1u << (pp - 1)) - 1u) & ~marked;   // earlier non-lost candidates
            if (!(r.y & 2u) || (r.y & 4u) || prior) break;   // check 2 fails or it breaks another deadline
            if ((r.x >> (pp - 1)) & 1u) marked |= 1u << (pp - 1);   // only its own deadline fails: lost
            adm = pp;
        }
    }
    n_adm[i] = adm;
    lost[i] = marked;
}

}  // namespace

int launch_admit_expand(const tp_inst* inst, int32_t n_inst, int32_t qc, const int32_t* n_adm1,
                        const uint32_t* status1, tp_inst* vinst, int32_t* vforce, cudaStream_t s) {
    const int64_t tot = (int64_t)n_inst * qc;
    if (tot == 0) return TP_OK;
    k_admit_expand<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(inst, n_inst, qc, n_adm1, status1, vinst, vforce);
    return cudaPeekAtLastError() == cudaSuccess ? TP_OK : TP_ECUDA;
}

int launch_admit_checks(const tp_inst* vinst, int32_t n_v, const tp_req* req, const double* t_dead,
                        const int32_t* vn, const uint32_t* vstatus, const K2Params& ws, int32_t H,
                        int64_t tbt_ticks, uint2* vres, cudaStream_t s) {
    if (n_v == 0) return TP_OK;
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return TP_ECUDA;
    const int max_bytes = kMaxHRunsSelect * 16 + (kMaxHRunsSelect + 1) * 4;
    if (H > kMaxHRunsSelect) return TP_EINVAL;
    if (dev < 64 && !done[dev]) {
        if (cudaFuncSetAttribute(k_admit_checks, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes) !=
            cudaSuccess)
            return TP_ECUDA;
        done[dev] = true;
    }
    CheckParams p{vinst, reinterpret_cast<const int4*>(req), t_dead, vn, vstatus, ws.run_h, ws.run_m, ws.run_key,
                  ws.cell_tab, ws.lut, H, (long long)tbt_ticks, vres};
    const size_t smem = (size_t)H * 16 + (size_t)(H + 1) * 4;
    k_admit_checks<<<n_v, kThreads, smem, s>>>(p);
    return cudaPeekAtLastError() == cudaSuccess ? TP_OK : TP_ECUDA;
}

int launch_admit_resolve(int32_t n_inst, int32_t qc, const tp_inst* inst, const uint32_t* status1,
                         const int32_t* n_adm1, const uint2* vres, int32_t* n_adm, uint32_t* lost, cudaStream_t s) {
    if (n_inst == 0) return TP_OK;
    k_admit_resolve<<<(n_inst + 127) / 128, 128, 0, s>>>(n_inst, qc, inst, status1, n_adm1, vres, n_adm, lost);
    return cudaPeekAtLastError() == cudaSuccess ? TP_OK : TP_ECUDA;
}

}  // namespace tp
