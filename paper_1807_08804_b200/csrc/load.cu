// load.cu -- a0: device-resident graph layout (P:630 nodes/edges arrays + label
// arrays; P:941 incoming + outgoing representations; P:679 freq(label)).
//
// Layout: off_out/off_in u32 [n+1]; arc_out/arc_in u32
// packed (dst << lbits) | elabel, each row sorted ascending (= by (dst, label))
// and de-duplicated (set semantics, reading R5); vlab u16 [n].  Undirected
// graphs are symmetrised and share one CSR for both directions.
#include <algorithm>

#include "prims.cuh"

namespace gps {

static inline int bitlen(uint64_t x) {
    int b = 0;
    while (x) {
        b++;
        x >>= 1;
    }
    return b;
}

// One thread per input arc: key = (src << pbits) | ((dst << lbits) | label).
__global__ void k_make_keys(const uint64_t* __restrict__ off, uint32_t n, const uint32_t* __restrict__ tgt,
                            const uint16_t* __restrict__ el, uint64_t m, uint32_t lbits, uint32_t pbits,
                            int undirected, uint64_t* __restrict__ keys) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    uint32_t lo = 0, hi = n;  // largest s with off[s] <= i
    while (hi - lo > 1) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (off[mid] <= i) lo = mid; else hi = mid;
    }
    uint64_t src = lo, dst = tgt[i], lab = el ? el[i] : 0;
    keys[i] = (src << pbits) | (dst << lbits) | lab;
    if (undirected) keys[m + i] = (dst << pbits) | (src << lbits) | lab;
}

__global__ void k_dup_flags(const uint64_t* __restrict__ keys, uint64_t m, uint32_t* __restrict__ flag) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

// Compact unique keys; write arc words and row offsets.
__global__ void k_build_rows(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ flag,
                             const uint32_t* __restrict__ pos, uint64_t m, uint32_t n, uint32_t pbits,
                             uint32_t total, uint32_t* __restrict__ arc, uint32_t* __restrict__ off,
                             uint64_t* __restrict__ ukeys) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint64_t pmask = (pbits >= 64) ? ~0ull : ((1ull << pbits) - 1);
    uint64_t k = keys[i];
    int64_t s = (int64_t)(k >> pbits);
    if (flag[i]) {
        uint32_t j = pos[i];
        arc[j] = (uint32_t)(k & pmask);
        if (ukeys) ukeys[j] = k;
        int64_t prev = i == 0 ? -1 : (int64_t)(keys[i - 1] >> pbits);
        for (int64_t v = prev + 1; v <= s; v++) off[v] = j;
    }
    if (i == m - 1)
        for (int64_t v = s + 1; v <= (int64_t)n; v++) off[v] = total;
}

__global__ void k_transpose_keys(const uint64_t* __restrict__ ukeys, uint64_t m, uint32_t lbits, uint32_t pbits,
                                 uint64_t* __restrict__ out) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint64_t pmask = (1ull << pbits) - 1;
    uint64_t k = ukeys[i];
    uint64_t src = k >> pbits, packed = k & pmask;
    uint64_t dst = packed >> lbits, lab = packed & ((1ull << lbits) - 1);
    out[i] = (dst << pbits) | (src << lbits) | lab;
}

__global__ void k_degrees(const uint32_t* __restrict__ off_out, const uint32_t* __restrict__ off_in, uint32_t n,
                          uint2* __restrict__ deg) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        deg[v] = make_uint2(off_out[v + 1] - off_out[v], off_in[v + 1] - off_in[v]);
}

__global__ void k_label_hist(const uint16_t* __restrict__ vlab, uint32_t n, uint32_t nl,
                             unsigned long long* __restrict__ hist) {
    extern __shared__ unsigned int s_h[];
    bool use_smem = nl <= 8192;
    if (use_smem)
        for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) s_h[i] = 0;
    __syncthreads();
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        if (use_smem) atomicAdd(&s_h[vlab[v]], 1u);
        else atomicAdd(&hist[vlab[v]], 1ull);
    }
    __syncthreads();
    if (use_smem)
        for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x)
            if (s_h[i]) atomicAdd(&hist[i], (unsigned long long)s_h[i]);
}

// Edge labels present in the stored arcs (f2 named variable edges bind only these):
// one bit per label value, OR-reduced in shared memory per block.
__global__ void k_elabel_set(const uint32_t* __restrict__ arcs, uint64_t m, uint32_t lmask,
                             unsigned int* __restrict__ bits) {
    __shared__ unsigned int s_b[2048];   // 2^16 labels at most
    const uint32_t nw = (lmask >> 5) + 1;
    for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x) s_b[i] = 0;
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t l = arcs[i] & lmask;
        atomicOr(&s_b[l >> 5], 1u << (l & 31));
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x)
        if (s_b[i]) atomicOr(&bits[i], s_b[i]);
}

// Sort + de-duplicate keys, emit one CSR direction.  Returns #unique arcs.
static uint32_t build_direction(gps_ctx* c, uint64_t* keys, uint64_t* tmp, uint64_t m, uint32_t n, uint32_t pbits,
                                int nbits, uint32_t* off, uint32_t** arc_out, uint64_t* ukeys_out) {
    radix_sort_u64(c, keys, tmp, m, nbits);
    DevPtr flag(c, sizeof(uint32_t) * (m + 1));
    DevPtr pos(c, sizeof(uint32_t) * (m + 1));
    const uint32_t T = 256;
    uint32_t g = (uint32_t)((m + T - 1) / T);
    launch(c, GPS_K_LOAD, dim3(g), dim3(T), 0, k_dup_flags, (const uint64_t*)keys, m, flag.as<uint32_t>());
    scan_exclusive1<uint32_t, uint32_t>(c, flag.as<uint32_t>(), pos.as<uint32_t>(), m);
    uint32_t total = 0;
    GPS_CK(cudaMemcpyAsync(&total, pos.as<uint32_t>() + m, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    ctx_sync(c);
    uint32_t* arc = static_cast<uint32_t*>(nullptr);
    GPS_CK(cudaMalloc(&arc, sizeof(uint32_t) * ((uint64_t)total + 4)));
    launch(c, GPS_K_LOAD, dim3(g), dim3(T), 0, k_build_rows, (const uint64_t*)keys, (const uint32_t*)flag.as<uint32_t>(),
           (const uint32_t*)pos.as<uint32_t>(), m, n, pbits, total, arc, off, ukeys_out);
    *arc_out = arc;
    return total;
}

void load_graph(gps_ctx* c, const gps_csr_desc* d, gps_graph* g) {
    if (!d) fail(GPS_EINVAL, "null graph descriptor");
    const uint32_t n = d->n_vertices;
    const uint64_t m = d->n_arcs;
    if (n == 0) fail(GPS_EINVAL, "graph with 0 vertices");
    if (!d->offsets || (m > 0 && !d->targets)) fail(GPS_EINVAL, "null offsets/targets");
    if (d->flags & ~GPS_UNDIRECTED) fail(GPS_EINVAL, "unknown graph flags");
    // ---- host validation (no arithmetic of the method: shape checks only) ----
    if (d->offsets[0] != 0 || d->offsets[n] != m) fail(GPS_EINVAL, "offsets[0] must be 0 and offsets[n] = n_arcs");
    for (uint32_t v = 0; v < n; v++)
        if (d->offsets[v + 1] < d->offsets[v]) fail(GPS_EINVAL, "offsets not non-decreasing");
    uint32_t maxel = 0;
    for (uint64_t i = 0; i < m; i++) {
        if (d->targets[i] >= n) fail(GPS_EINVAL, "target >= n_vertices");
        if (d->edge_labels && d->edge_labels[i] > maxel) maxel = d->edge_labels[i];
    }
    uint32_t maxvl = 0;
    if (d->vertex_labels)
        for (uint32_t v = 0; v < n; v++) maxvl = std::max<uint32_t>(maxvl, d->vertex_labels[v]);
    const bool und = (d->flags & GPS_UNDIRECTED) != 0;
    const uint32_t lbits = (uint32_t)bitlen(maxel);
    const uint32_t pbits = (uint32_t)bitlen((uint64_t)(n - 1)) + lbits;
    if (pbits > 32) fail(GPS_EUNSUPPORTED, "(n-1) << label_bits does not fit 32 bits");
    const uint64_t mk = und ? 2 * m : m;
    if (mk >= (1ull << 32)) fail(GPS_EUNSUPPORTED, ">= 2^32 arcs");
    const int nbits = bitlen((uint64_t)(n - 1)) + (int)pbits;

    g->d.n = n;
    g->d.nw = (n + 31) / 32;
    g->d.nws = ((g->d.nw + 63) / 64) * 64;
    g->d.lbits = lbits;
    g->d.lmask = lbits ? ((1u << lbits) - 1u) : 0u;
    g->undirected = und;
    g->n_vlabels = maxvl + 1;

    // ---- upload inputs (stream-ordered scratch) ----
    DevPtr doff(c, sizeof(uint64_t) * (n + 1));
    DevPtr dtgt(c, sizeof(uint32_t) * (m + 1));
    DevPtr del(c, d->edge_labels ? sizeof(uint16_t) * (m + 1) : 16);
    GPS_CK(cudaMemcpyAsync(doff.p, d->offsets, sizeof(uint64_t) * (n + 1), cudaMemcpyHostToDevice, c->stream));
    if (m) GPS_CK(cudaMemcpyAsync(dtgt.p, d->targets, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, c->stream));
    if (m && d->edge_labels)
        GPS_CK(cudaMemcpyAsync(del.p, d->edge_labels, sizeof(uint16_t) * m, cudaMemcpyHostToDevice, c->stream));

    uint32_t *off_out = nullptr, *off_in = nullptr, *arc_out = nullptr, *arc_in = nullptr;
    uint16_t* vlab = nullptr;
    GPS_CK(cudaMalloc(&off_out, sizeof(uint32_t) * (n + 1)));
    g->mem[0] = off_out;
    GPS_CK(cudaMemsetAsync(off_out, 0, sizeof(uint32_t) * (n + 1), c->stream));
    DevPtr keys(c, sizeof(uint64_t) * (mk + 1));
    DevPtr tmp(c, sizeof(uint64_t) * (mk + 1));
    DevPtr ukeys(c, sizeof(uint64_t) * (mk + 1));
    const uint32_t T = 256;
    if (m)
        launch(c, GPS_K_LOAD, dim3((uint32_t)((m + T - 1) / T)), dim3(T), 0, k_make_keys,
               (const uint64_t*)doff.as<uint64_t>(), n, (const uint32_t*)dtgt.as<uint32_t>(),
               (const uint16_t*)(d->edge_labels ? del.as<uint16_t>() : nullptr), m, lbits, pbits, und ? 1 : 0,
               keys.as<uint64_t>());
    uint32_t mu = 0;
    if (mk) {
        mu = build_direction(c, keys.as<uint64_t>(), tmp.as<uint64_t>(), mk, n, pbits, nbits, off_out, &arc_out,
                             und ? nullptr : ukeys.as<uint64_t>());
    } else {
        GPS_CK(cudaMalloc(&arc_out, 16));
    }
    g->mem[1] = arc_out;
    g->m = mu;
    if (und) {
        off_in = off_out;
        arc_in = arc_out;
    } else {
        GPS_CK(cudaMalloc(&off_in, sizeof(uint32_t) * (n + 1)));
        g->mem[2] = off_in;
        GPS_CK(cudaMemsetAsync(off_in, 0, sizeof(uint32_t) * (n + 1), c->stream));
        if (mu) {
            launch(c, GPS_K_LOAD, dim3((mu + T - 1) / T), dim3(T), 0, k_transpose_keys,
                   (const uint64_t*)ukeys.as<uint64_t>(), (uint64_t)mu, lbits, pbits, keys.as<uint64_t>());
            uint32_t mi = build_direction(c, keys.as<uint64_t>(), tmp.as<uint64_t>(), mu, n, pbits, nbits, off_in,
                                          &arc_in, nullptr);
            if (mi != mu) fail(GPS_ECUDA, "incoming CSR size mismatch");
        } else {
            GPS_CK(cudaMalloc(&arc_in, 16));
        }
        g->mem[3] = arc_in;
    }
    GPS_CK(cudaMalloc(&vlab, sizeof(uint16_t) * (n + 8)));
    g->mem[4] = vlab;
    if (d->vertex_labels)
        GPS_CK(cudaMemcpyAsync(vlab, d->vertex_labels, sizeof(uint16_t) * n, cudaMemcpyHostToDevice, c->stream));
    else
        GPS_CK(cudaMemsetAsync(vlab, 0, sizeof(uint16_t) * n, c->stream));
    // freq(label) histogram, computed on the device
    DevPtr dh(c, sizeof(unsigned long long) * g->n_vlabels);
    GPS_CK(cudaMemsetAsync(dh.p, 0, sizeof(unsigned long long) * g->n_vlabels, c->stream));
    size_t smem = g->n_vlabels <= 8192 ? g->n_vlabels * sizeof(unsigned int) : 0;
    launch(c, GPS_K_LOAD, dim3(std::min<uint32_t>((n + 255) / 256, 1184)), dim3(256), smem, k_label_hist,
           (const uint16_t*)vlab, n, g->n_vlabels, dh.as<unsigned long long>());
    std::vector<unsigned long long> h(g->n_vlabels);
    GPS_CK(cudaMemcpyAsync(h.data(), dh.p, sizeof(unsigned long long) * g->n_vlabels, cudaMemcpyDeviceToHost,
                           c->stream));
    const uint32_t elw = (g->d.lmask >> 5) + 1;
    DevPtr del_bits(c, sizeof(unsigned int) * elw);
    GPS_CK(cudaMemsetAsync(del_bits.p, 0, sizeof(unsigned int) * elw, c->stream));
    if (mu)
        launch(c, GPS_K_LOAD, dim3(std::min<uint32_t>((mu + 255) / 256, 1184)), dim3(256), 0, k_elabel_set,
               (const uint32_t*)arc_out, (uint64_t)mu, g->d.lmask, del_bits.as<unsigned int>());
    std::vector<unsigned int> elb(elw);
    GPS_CK(cudaMemcpyAsync(elb.data(), del_bits.p, sizeof(unsigned int) * elw, cudaMemcpyDeviceToHost, c->stream));
    uint2* deg = nullptr;
    GPS_CK(cudaMalloc(&deg, sizeof(uint2) * (n + 1)));
    g->mem[5] = deg;
    if (n)
        launch(c, GPS_K_LOAD, dim3(std::min<uint32_t>((n + 255) / 256, 4096)), dim3(256), 0, k_degrees,
               (const uint32_t*)off_out, (const uint32_t*)off_in, n, deg);
    ctx_sync(c);
    g->lab_hist.assign(h.begin(), h.end());
    g->elabels.clear();
    for (uint32_t l = 0; l <= g->d.lmask; l++)
        if ((elb[l >> 5] >> (l & 31)) & 1u) g->elabels.push_back(l);
    g->d.off_out = off_out;
    g->d.arc_out = arc_out;
    g->d.off_in = off_in;
    g->d.arc_in = arc_in;
    g->d.vlab = vlab;
    g->d.deg = deg;
}

void free_graph_mem(gps_graph* g) {
    for (void*& p : g->mem) {
        if (p) cudaFree(p);
        p = nullptr;
    }
}

}  // namespace gps
