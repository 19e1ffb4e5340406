// tp_gbdt_load / tp_gbdt_free: parse blob v1 (include/tp.h), validate, normalise to the
// complete-heap, rank-encoded node words K2 streams through shared memory, upload.
//
// The model is the paper's performance model M (PAPER §4.3.1): a gradient-boosted
// tree ensemble over [engine size, batch, KV usage, GPU frequency] predicting IPS.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <vector>

#include "tp_internal.cuh"

namespace {

struct Node {
    int32_t feature;
    float threshold;
    int32_t left, right;
    float leaf;
};

uint32_t rd32(const unsigned char* p) {
    uint32_t v;
    std::memcpy(&v, p, 4);
    return v;
}

// depth-first validation: indices in range, every node reached exactly once (no cycle or
// sharing), feature in [-1, 3], finite values, depth bound.  Returns max depth or -1.
int validate(const std::vector<Node>& t, int at, int depth, int max_depth, std::vector<char>& seen) {
    if (at < 0 || at >= (int)t.size() || seen[at]) return -1;
    seen[at] = 1;
    const Node& nd = t[at];
    if (nd.feature == -1) {
        if (!std::isfinite(nd.leaf) || std::fabs(nd.leaf) > 0x1p60f) return -1;
        return depth;
    }
    if (nd.feature < 0 || nd.feature > 3 || !std::isfinite(nd.threshold)) return -1;
    if (depth + 1 > max_depth) return -1;
    int a = validate(t, nd.left, depth + 1, max_depth, seen);
    if (a < 0) return -1;
    int b = validate(t, nd.right, depth + 1, max_depth, seen);
    if (b < 0) return -1;
    return std::max(a, b);
}

uint32_t sel_of(int f) {
    uint32_t b0 = 2u * f, b1 = 2u * f + 1u;
    return b1 | (b1 << 4) | (b0 << 8) | (b1 << 12);
}

void fill(const std::vector<Node>& t, int at, uint32_t idx, int depth, int D,
          const std::vector<float> (&cuts)[4], uint32_t* w) {
    const Node& nd = t[at];
    if (depth == D) {                 // leaf level of the complete heap
        uint32_t bits;
        std::memcpy(&bits, &nd.leaf, 4);
        w[idx] = bits;
        return;
    }
    if (nd.feature == -1) {           // shallow leaf: always-left word, replicate the leaf below
        w[idx] = (0x8000u << 16) | sel_of(0);   // rank <= 0x7FFF never exceeds j = 0x7FFF
        fill(t, at, 2 * idx, depth + 1, D, cuts, w);
        fill(t, at, 2 * idx + 1, depth + 1, D, cuts, w);
        return;
    }
    const std::vector<float>& c = cuts[nd.feature];
    // index of the threshold among the feature's distinct cuts (fp32 equality: -0 == +0)
    auto it = std::lower_bound(c.begin(), c.end(), nd.threshold);
    uint32_t j = (uint32_t)(it - c.begin());
    w[idx] = ((0xFFFFu - j) << 16) | sel_of(nd.feature);
    fill(t, nd.left, 2 * idx, depth + 1, D, cuts, w);
    fill(t, nd.right, 2 * idx + 1, depth + 1, D, cuts, w);
}

}  // namespace

namespace {
int load_impl(const void* host_blob, size_t nbytes, int device, tp_gbdt** out) {
    const unsigned char* p = (const unsigned char*)host_blob;
    if (nbytes < 24 || std::memcmp(p, "TPGB", 4) != 0) return TP_EFORMAT;
    if (rd32(p + 4) != 1 || rd32(p + 8) != 4) return TP_EFORMAT;
    uint32_t nt = rd32(p + 12), md = rd32(p + 16);
    float base;
    std::memcpy(&base, p + 20, 4);
    if (nt > (1u << 20) || md > (uint32_t)tp::kMaxDepth || !std::isfinite(base)) return TP_EFORMAT;

    std::vector<std::vector<Node>> trees(nt);
    size_t off = 24;
    int D = 0;
    for (uint32_t t = 0; t < nt; ++t) {
        if (off + 4 > nbytes) return TP_EFORMAT;
        uint32_t c = rd32(p + off);
        off += 4;
        if (c < 1 || c > 8192u || off + (size_t)c * 20 > nbytes) return TP_EFORMAT;
        trees[t].resize(c);
        for (uint32_t i = 0; i < c; ++i, off += 20) std::memcpy(&trees[t][i], p + off, 20);
        std::vector<char> seen(c, 0);
        int d = validate(trees[t], 0, 0, (int)md, seen);
        if (d < 0) return TP_EFORMAT;
        for (uint32_t i = 0; i < c; ++i)
            if (!seen[i]) return TP_EFORMAT;   // unreachable node
        D = std::max(D, d);
    }
    if (off != nbytes) return TP_EFORMAT;

    // distinct thresholds per feature, ascending (the rank encoding's cut lists)
    std::vector<float> cuts[4];
    for (auto& t : trees)
        for (auto& nd : t)
            if (nd.feature >= 0) cuts[nd.feature].push_back(nd.threshold == 0.f ? 0.f : nd.threshold);
    for (int f = 0; f < 4; ++f) {
        std::sort(cuts[f].begin(), cuts[f].end());
        cuts[f].erase(std::unique(cuts[f].begin(), cuts[f].end()), cuts[f].end());
        if ((int)cuts[f].size() > tp::kMaxCuts) return TP_EFORMAT;
    }

    // Output range of the ensemble: base + sum over trees of [min leaf, max leaf], widened by a bound
    // on the fp32 rounding of the sequential sum (each addition errs by <= 2^-24 of a partial sum
    // whose magnitude is <= S).  If every output is inside (1, 512) IPS, T' = fl32(1/ips) lies in
    // (2^-9, 1) s for every cell and level: its tick count (units of 2^-40 s) is a multiple of 2^8
    // below 2^40, so the compact path keeps T' / 2^8 ticks in 32 bits, exactly (tick_shift = 8).
    double out_lo = base, out_hi = base, S = std::fabs((double)base);
    for (auto& t : trees) {
        double mn = INFINITY, mx = -INFINITY;
        for (auto& nd : t)
            if (nd.feature == -1) {
                mn = std::min(mn, (double)nd.leaf);
                mx = std::max(mx, (double)nd.leaf);
            }
        out_lo += mn;
        out_hi += mx;
        S += std::max(std::fabs(mn), std::fabs(mx));
    }
    const double rerr = 2.0 * ((double)nt + 1.0) * 0x1p-24 * S;
    const int tick_shift = (out_lo - rerr > 1.0 && out_hi + rerr < 512.0) ? 8 : 0;

    const size_t words_per_tree = std::max<size_t>(4, (size_t)2 << D);   // >= 16 B: TMA size/alignment unit
    if ((uint64_t)nt * words_per_tree > tp::kMaxModelWords) return TP_EFORMAT;  // > 1 GiB of node words
    std::vector<uint32_t> words(std::max<size_t>(1, nt * words_per_tree), 0u);
    for (uint32_t t = 0; t < nt; ++t) fill(trees[t], 0, 1u, 0, D, cuts, &words[t * words_per_tree]);
    std::vector<float> allc;
    tp_gbdt* h = new (std::nothrow) tp_gbdt();
    if (!h) return TP_ENOMEM;
    tp::Model& m = h->m;
    m.device = device;
    m.n_trees = (int32_t)nt;
    m.depth = D;
    m.base = base;
    m.tick_shift = tick_shift;
    for (int f = 0; f < 4; ++f) {
        m.n_cuts[f] = (int32_t)cuts[f].size();
        m.cut_off[f] = (int32_t)allc.size();
        allc.insert(allc.end(), cuts[f].begin(), cuts[f].end());
    }
    m.cut_off[4] = (int32_t)allc.size();
    allc.push_back(0.f);   // never empty
    // rank tables for integer batch / KV values: rank(x) = #cuts <= x for x in [0, len).  The table
    // runs one past the largest cut (len = floor(max cut) + 2, at least 1), so its last entry is
    // the rank of every larger x too: rank(x) = rtab[min(x, len - 1)] for every x >= 0 unless the
    // table is capped at kRankTabMax entries (then exact for x < kRankTabMax).
    std::vector<uint16_t> rtab;
    for (int w = 0; w < 2; ++w) {
        const std::vector<float>& c = cuts[1 + w];
        int64_t len = 1;
        if (!c.empty() && c.back() >= 0.f) len = std::min<int64_t>((int64_t)std::floor(c.back()) + 2, tp::kRankTabMax);
        m.rtab_off[w] = (int32_t)rtab.size();
        m.rtab_len[w] = (int32_t)len;
        for (int64_t x = 0; x < len; ++x)
            rtab.push_back((uint16_t)(std::upper_bound(c.begin(), c.end(), (float)x) - c.begin()));
    }
    rtab.push_back(0);
    while (rtab.size() % 8) rtab.push_back(0);   // whole 16-byte words (K1c copies the tables to shared memory in 32-bit words)

    int prev = 0;
    if (cudaGetDevice(&prev) != cudaSuccess || cudaSetDevice(device) != cudaSuccess) {
        delete h;
        return TP_ECUDA;
    }
    int rc = TP_OK;
    size_t wb = words.size() * 4, cb = allc.size() * 4, rb = rtab.size() * 2;
    if (cudaMalloc(&m.d_words, wb) != cudaSuccess || cudaMalloc(&m.d_cuts, cb) != cudaSuccess ||
        cudaMalloc(&m.d_rtab, rb) != cudaSuccess) {
        rc = TP_ENOMEM;
    } else if (cudaMemcpy(m.d_words, words.data(), wb, cudaMemcpyHostToDevice) != cudaSuccess ||
               cudaMemcpy(m.d_cuts, allc.data(), cb, cudaMemcpyHostToDevice) != cudaSuccess ||
               cudaMemcpy(m.d_rtab, rtab.data(), rb, cudaMemcpyHostToDevice) != cudaSuccess) {
        rc = TP_ECUDA;
    }
    m.device_bytes = (int64_t)(wb + cb + rb);
    cudaSetDevice(prev);
    if (rc != TP_OK) {
        tp_gbdt_free(h);
        return rc;
    }
    *out = h;
    return TP_OK;
}
}  // namespace

// The parse allocates host vectors sized from the blob: an allocation failure must not cross
// the C ABI as an exception (it would terminate the caller), so it becomes TP_ENOMEM.
extern "C" int tp_gbdt_load(const void* host_blob, size_t nbytes, int device, tp_gbdt** out) {
    if (!host_blob || !out) return TP_EINVAL;
    *out = nullptr;
    try {
        return load_impl(host_blob, nbytes, device, out);
    } catch (const std::bad_alloc&) {
        return TP_ENOMEM;
    } catch (...) {
        return TP_EFORMAT;
    }
}

extern "C" int tp_gbdt_free(tp_gbdt* h) {
    if (!h) return TP_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(h->m.device);
    if (h->m.d_words) cudaFree(h->m.d_words);
    if (h->m.d_cuts) cudaFree(h->m.d_cuts);
    if (h->m.d_rtab) cudaFree(h->m.d_rtab);
    cudaSetDevice(prev);
    delete h;
    return TP_OK;
}

extern "C" int tp_gbdt_get_info(const tp_gbdt* h, tp_gbdt_info* out) {
    if (!h || !out) return TP_EINVAL;
    std::memset(out, 0, sizeof(*out));
    out->n_trees = h->m.n_trees;
    out->depth = h->m.depth;
    for (int f = 0; f < 4; ++f) out->n_cuts[f] = h->m.n_cuts[f];
    out->base_score = h->m.base;
    out->tick_shift = h->m.tick_shift;
    out->device_bytes = h->m.device_bytes;
    out->node_bytes = (int64_t)h->m.n_trees * std::max<int64_t>(4, (int64_t)2 << h->m.depth) * 4;
    return TP_OK;
}
