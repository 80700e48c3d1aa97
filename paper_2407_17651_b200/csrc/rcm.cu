// Reverse Cuthill-McKee on the GPU, bit-identical to
// the reference's rcm_order (reorder.py:137-286) and to the host-native
// version in prep.cpp.
//
// Every component is processed at once, in lockstep, by level-synchronous
// multi-source BFS (components are disjoint, so one frontier carries all of
// them):
//   1. components: min-label hooking + pointer jumping gives each node the
//      smallest index of its component (its root); the reference visits
//      components in that order and appends isolated nodes in scan order,
//      so component c's block of positions starts at the number of nodes
//      whose root is smaller;
//   2. start nodes: the min-(degree, index) member of each component, then
//      the George-Liu walk (reorder.py:234-248): BFS from the current
//      candidate, move to the min-(degree, index) node of the deepest level
//      while the eccentricity grows -- one multi-source BFS per round for
//      all components still walking;
//   3. Cuthill-McKee: level L+1 of a component, sorted by (position of its
//      minimum-position level-L neighbour, degree, index), is the
//      reference's queue order (prep.cpp has the argument); each level is
//      expanded by one kernel, sorted with two stable CUB radix sorts (index,
//      then (parent position, degree)) and placed after the component's
//      previous levels;
//   4. reverse: forward[v] = n - 1 - position[v].
// The adjacency can be given as a pattern (indptr/indices, any neighbour
// order) or built on the device from the strictly-lower SSS arrays.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <cstdint>
#include <vector>

#include "common.h"

namespace {

constexpr int kTB = 256;
constexpr unsigned long long kInf = ~0ull;

inline int blocks_for(int64_t n) { return (int)std::min<int64_t>((n + kTB - 1) / kTB, 148 * 64); }

template <class T>
struct DevBuf {
    T *p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t count) { return cudaMalloc((void **)&p, sizeof(T) * (count ? count : 1)); }
};

// ---- adjacency from the strictly-lower SSS arrays ------------------------
__global__ void k_deg_lower(int64_t n, const int64_t *rp, const int32_t *ci, int64_t *cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        atomicAdd((unsigned long long *)&cnt[i], (unsigned long long)(rp[i + 1] - rp[i]));
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) atomicAdd((unsigned long long *)&cnt[ci[k]], 1ull);
    }
}

__global__ void k_fill_lower(int64_t n, const int64_t *rp, const int32_t *ci, int64_t *fill,
                             int32_t *idx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t nl = rp[i + 1] - rp[i];
        const int64_t o = atomicAdd((unsigned long long *)&fill[i], (unsigned long long)nl);
        for (int64_t k = 0; k < nl; k++) {
            const int32_t c = ci[rp[i] + k];
            idx[o + k] = c;
            idx[atomicAdd((unsigned long long *)&fill[c], 1ull)] = (int32_t)i;
        }
    }
}

// ---- components -----------------------------------------------------------
__global__ void k_iota(int64_t n, int32_t *a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int32_t)i;
}

__device__ __forceinline__ int32_t find_root(const int32_t *lab, int32_t u) {
    int32_t r = lab[u];
    while (true) {
        const int32_t q = lab[r];
        if (q == r) return r;
        r = q;
    }
}

// hook (ECL-CC style): every edge links the two trees, the larger root
// under the smaller one with a CAS that only succeeds on a root, so the
// final root of each tree is the smallest index of its component
__global__ void k_hook(int64_t n, const int64_t *ip, const int32_t *ix, int32_t *lab) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        for (int64_t k = ip[u]; k < ip[u + 1]; k++) {
            const int32_t w = ix[k];
            if (w <= u) continue;  // each undirected edge once
            while (true) {
                const int32_t a = find_root(lab, (int32_t)u), b = find_root(lab, w);
                if (a == b) break;
                const int32_t hi = a > b ? a : b, lo = a ^ b ^ hi;
                if (atomicCAS(&lab[hi], hi, lo) == hi) break;
            }
        }
    }
}

__global__ void k_compress(int64_t n, int32_t *lab) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        lab[u] = find_root(lab, (int32_t)u);
}

// ---- start candidates -------------------------------------------------------
__device__ __forceinline__ unsigned long long dkey(int64_t deg, int32_t u) {
    return ((unsigned long long)deg << 32) | (uint32_t)u;
}

__global__ void k_min_member(int64_t n, const int64_t *ip, const int32_t *root, unsigned long long *best) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        atomicMin(&best[root[u]], dkey(ip[u + 1] - ip[u], (int32_t)u));
}

// ---- multi-source BFS (George-Liu rounds) ---------------------------------
__global__ void k_expand_bfs(const int32_t *front, int f, const int64_t *ip, const int32_t *ix,
                             int32_t *level, int32_t lvl, int32_t *next, int *ncount) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < f; t += gridDim.x * blockDim.x) {
        const int32_t u = front[t];
        for (int64_t k = ip[u]; k < ip[u + 1]; k++) {
            const int32_t w = ix[k];
            if (level[w] < 0 && atomicCAS(&level[w], -1, lvl) == -1) next[atomicAdd(ncount, 1)] = w;
        }
    }
}

// per component: eccentricity = deepest level, then min (degree, index) there
__global__ void k_ecc(const int32_t *visited, int nv, const int32_t *level, const int32_t *root,
                      int32_t *ecc) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nv; t += gridDim.x * blockDim.x) {
        const int32_t u = visited[t];
        atomicMax(&ecc[root[u]], level[u]);
    }
}

__global__ void k_deepest(const int32_t *visited, int nv, const int32_t *level, const int32_t *root,
                          const int32_t *ecc, const int64_t *ip, unsigned long long *best) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nv; t += gridDim.x * blockDim.x) {
        const int32_t u = visited[t];
        const int32_t c = root[u];
        if (level[u] == ecc[c]) atomicMin(&best[c], dkey(ip[u + 1] - ip[u], u));
    }
}

__global__ void k_reset_level(const int32_t *visited, int nv, int32_t *level) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nv; t += gridDim.x * blockDim.x) level[visited[t]] = -1;
}

// George-Liu step per walking component c (active[c] != 0), after BFS(y):
// ecc_y > ecc_x -> x = y, ecc_x = ecc_y, y = z (keep walking), else stop
__global__ void k_walk(const int32_t *comps, int ncomp, int32_t *cand_x, int32_t *ecc_x, int32_t *cand_y,
                       const int32_t *ecc, const unsigned long long *best, int32_t *active, int *nactive,
                       int first) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ncomp; t += gridDim.x * blockDim.x) {
        const int32_t c = comps[t];
        if (!active[c]) continue;
        const int32_t z = (int32_t)(best[c] & 0xffffffffu);
        if (first) {  // BFS was from x
            ecc_x[c] = ecc[c];
            cand_y[c] = z;
            atomicAdd(nactive, 1);
        } else if (ecc[c] > ecc_x[c]) {
            cand_x[c] = cand_y[c];
            ecc_x[c] = ecc[c];
            cand_y[c] = z;
            atomicAdd(nactive, 1);
        } else {
            active[c] = 0;
        }
    }
}

// ---- Cuthill-McKee placement ---------------------------------------------
__global__ void k_expand_cm(const int32_t *front, int f, const int64_t *ip, const int32_t *ix,
                            const int64_t *pos, unsigned long long *parent, int32_t *next, int *ncount) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < f; t += gridDim.x * blockDim.x) {
        const int32_t u = front[t];
        const unsigned long long pu = (unsigned long long)pos[u];
        for (int64_t k = ip[u]; k < ip[u + 1]; k++) {
            const int32_t w = ix[k];
            if (pos[w] >= 0) continue;
            if (atomicMin(&parent[w], pu) == kInf) next[atomicAdd(ncount, 1)] = w;  // first visitor
        }
    }
}

__global__ void k_cm_key(const int32_t *nodes, int f, const unsigned long long *parent, const int64_t *ip,
                         unsigned long long *key) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < f; t += gridDim.x * blockDim.x) {
        const int32_t w = nodes[t];
        key[t] = (parent[w] << 32) | (unsigned long long)(ip[w + 1] - ip[w]);
    }
}

// sorted level: node t of component c takes next_free[c] + (t - start of c's run)
__global__ void k_place(const int32_t *nodes, int f, const int32_t *root, int64_t *pos, int64_t *next_free) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < f; t += gridDim.x * blockDim.x) {
        const int32_t w = nodes[t];
        const int32_t c = root[w];
        int s = t;  // run start: runs are short except in one giant component; binary search back
        int lo = 0, hi = t;
        while (lo < hi) {  // first index in [0, t] whose component is c (components contiguous)
            const int mid = (lo + hi) >> 1;
            if (root[nodes[mid]] == c) hi = mid;
            else lo = mid + 1;
        }
        s = lo;
        pos[w] = next_free[c] + (t - s);
    }
}

__global__ void k_advance(const int32_t *nodes, int f, const int32_t *root, int64_t *next_free) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < f; t += gridDim.x * blockDim.x) {
        const int32_t c = root[nodes[t]];
        if (t + 1 == f || root[nodes[t + 1]] != c) {  // last of c's run
            int lo = 0, hi = t;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (root[nodes[mid]] == c) hi = mid;
                else lo = mid + 1;
            }
            next_free[c] += (t - lo + 1);
        }
    }
}

__global__ void k_root_count(int64_t n, const int32_t *root, int64_t *cnt) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long *)&cnt[root[u]], 1ull);
}

// roots of non-isolated components, and the isolated nodes' final positions
__global__ void k_seed(int64_t n, const int64_t *ip, const int32_t *root, const int64_t *base,
                       const unsigned long long *best, int64_t *pos, int32_t *comps, int *ncomp) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        if (ip[u + 1] == ip[u]) {
            pos[u] = base[u];  // isolated: its own block (root == u)
        } else if (root[u] == (int32_t)u) {
            comps[atomicAdd(ncomp, 1)] = (int32_t)u;
        }
        (void)best;
    }
}

__global__ void k_sources(const int32_t *comps, int ncomp, const int32_t *src, const int32_t *active,
                          int32_t *front, int *fcount, int32_t *level) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ncomp; t += gridDim.x * blockDim.x) {
        const int32_t c = comps[t];
        if (active && !active[c]) continue;
        const int32_t s = src[c];
        level[s] = 0;
        front[atomicAdd(fcount, 1)] = s;
    }
}

__global__ void k_cm_start(const int32_t *comps, int ncomp, const int32_t *start, const int64_t *base,
                           int64_t *pos, int64_t *next_free, int32_t *front) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ncomp; t += gridDim.x * blockDim.x) {
        const int32_t c = comps[t];
        const int32_t s = start[c];
        pos[s] = base[c];
        next_free[c] = base[c] + 1;
        front[t] = s;
    }
}

__global__ void k_forward(int64_t n, const int64_t *pos, int64_t *forward) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        forward[u] = n - 1 - pos[u];
}

__global__ void k_best_lo(const int32_t *comps, int ncomp, const unsigned long long *best, int32_t *out) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ncomp; t += gridDim.x * blockDim.x) {
        const int32_t c = comps[t];
        out[c] = (int32_t)(best[c] & 0xffffffffu);
    }
}

int bits_for(int64_t v) {
    int b = 1;
    while (b < 64 && (1ll << b) <= v) b++;
    return b;
}

#define RC(expr)                                                                                  \
    do {                                                                                          \
        cudaError_t _e = (expr);                                                                  \
        if (_e != cudaSuccess) PARS3_FAIL(PARS3_ERR_CUDA, "rcm_order_device: %s: %s", #expr,    \
                                          cudaGetErrorString(_e));                               \
    } while (0)

int read_int(const int *d, int *h, cudaStream_t st) {
    RC(cudaMemcpyAsync(h, d, sizeof(int), cudaMemcpyDeviceToHost, st));
    RC(cudaStreamSynchronize(st));
    return PARS3_OK;
}

// multi-source BFS from the sources already at vis[0, *nvis) (levels 0):
// every level is appended to `vis`, so on return vis[0, *nvis) is the
// visited set
int bfs(const int64_t *ip, const int32_t *ix, int32_t *level, int32_t *vis, int *nvis, int *d_cnt,
        cudaStream_t st) {
    int64_t a = 0, b = *nvis;
    int32_t lvl = 0;
    while (b > a) {
        RC(cudaMemsetAsync(d_cnt, 0, sizeof(int), st));
        lvl++;
        k_expand_bfs<<<blocks_for(b - a), kTB, 0, st>>>(vis + a, (int)(b - a), ip, ix, level, lvl,
                                                        vis + b, d_cnt);
        RC(cudaGetLastError());
        int fn = 0;
        if (int rc = read_int(d_cnt, &fn, st)) return rc;
        a = b;
        b += fn;
    }
    *nvis = (int)b;
    return PARS3_OK;
}

}  // namespace

namespace {

__global__ void k_fill_i32(int64_t n, int32_t *a, int32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}

__global__ void k_comp_reset(const int32_t *comps, int ncomp, const int32_t *active, int32_t *ecc,
                             unsigned long long *best) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ncomp; t += gridDim.x * blockDim.x) {
        const int32_t c = comps[t];
        if (active[c]) {
            ecc[c] = 0;
            best[c] = kInf;
        }
    }
}

__global__ void k_activate(const int32_t *comps, int ncomp, int32_t *active) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ncomp; t += gridDim.x * blockDim.x) active[comps[t]] = 1;
}

int rcm_device(int64_t n, const int64_t *ip, const int32_t *ix, int64_t *forward, cudaStream_t st) {
    if (n == 0) return PARS3_OK;
    DevBuf<int32_t> root, level, vis, comps, cand_x, cand_y, ecc_x, ecc, active, tmp;
    DevBuf<int64_t> cnt, base, pos, next_free;
    DevBuf<unsigned long long> best, parent, key, key_alt;
    DevBuf<int> d_cnt;
    RC(root.alloc(n));
    RC(level.alloc(n));
    RC(vis.alloc(n));
    RC(comps.alloc(n));
    RC(cand_x.alloc(n));
    RC(cand_y.alloc(n));
    RC(ecc_x.alloc(n));
    RC(ecc.alloc(n));
    RC(active.alloc(n));
    RC(tmp.alloc(n));
    RC(cnt.alloc(n));
    RC(base.alloc(n));
    RC(pos.alloc(n));
    RC(next_free.alloc(n));
    RC(best.alloc(n));
    RC(parent.alloc(n));
    RC(key.alloc(n));
    RC(key_alt.alloc(n));
    RC(d_cnt.alloc(2));
    const int G = blocks_for(n);
    // 1. components (root = smallest index)
    k_iota<<<G, kTB, 0, st>>>(n, root.p);
    k_hook<<<G, kTB, 0, st>>>(n, ip, ix, root.p);
    k_compress<<<G, kTB, 0, st>>>(n, root.p);
    // 2. block bases: base[r] = nodes whose root is below r
    RC(cudaMemsetAsync(cnt.p, 0, sizeof(int64_t) * n, st));
    k_root_count<<<G, kTB, 0, st>>>(n, root.p, cnt.p);
    size_t tb_scan = 0, tb_s1 = 0, tb_s2 = 0;
    RC(cub::DeviceScan::ExclusiveSum(nullptr, tb_scan, cnt.p, base.p, n, st));
    RC(cub::DeviceRadixSort::SortKeys(nullptr, tb_s1, vis.p, tmp.p, (int)n, 0, 32, st));
    RC(cub::DeviceRadixSort::SortPairs(nullptr, tb_s2, key.p, key_alt.p, tmp.p, vis.p, (int)n, 0, 64, st));
    DevBuf<uint8_t> temp;
    const size_t tb = std::max(tb_scan, std::max(tb_s1, tb_s2));
    RC(temp.alloc(tb));
    size_t t0 = tb;
    RC(cub::DeviceScan::ExclusiveSum(temp.p, t0, cnt.p, base.p, n, st));
    // 3. isolated nodes placed; non-isolated component roots listed
    RC(cudaMemsetAsync(pos.p, 0xff, sizeof(int64_t) * n, st));
    RC(cudaMemsetAsync(d_cnt.p, 0, sizeof(int) * 2, st));
    k_seed<<<G, kTB, 0, st>>>(n, ip, root.p, base.p, best.p, pos.p, comps.p, d_cnt.p);
    RC(cudaGetLastError());
    int ncomp = 0;
    if (int rc = read_int(d_cnt.p, &ncomp, st)) return rc;
    if (ncomp > 0) {
        const int GC = blocks_for(ncomp);
        // 4. George-Liu start per component, all components in lockstep
        RC(cudaMemsetAsync(best.p, 0xff, sizeof(unsigned long long) * n, st));
        k_min_member<<<G, kTB, 0, st>>>(n, ip, root.p, best.p);
        k_best_lo<<<GC, kTB, 0, st>>>(comps.p, ncomp, best.p, cand_x.p);
        RC(cudaMemsetAsync(active.p, 0, sizeof(int32_t) * n, st));
        k_activate<<<GC, kTB, 0, st>>>(comps.p, ncomp, active.p);
        k_fill_i32<<<G, kTB, 0, st>>>(n, level.p, -1);
        for (int first = 1;; first = 0) {
            RC(cudaMemsetAsync(d_cnt.p, 0, sizeof(int), st));
            k_sources<<<GC, kTB, 0, st>>>(comps.p, ncomp, first ? cand_x.p : cand_y.p, active.p, vis.p,
                                          d_cnt.p, level.p);
            RC(cudaGetLastError());
            int nvis = 0;
            if (int rc = read_int(d_cnt.p, &nvis, st)) return rc;
            if (int rc = bfs(ip, ix, level.p, vis.p, &nvis, d_cnt.p, st)) return rc;
            k_comp_reset<<<GC, kTB, 0, st>>>(comps.p, ncomp, active.p, ecc.p, best.p);
            const int GV = blocks_for(nvis);
            k_ecc<<<GV, kTB, 0, st>>>(vis.p, nvis, level.p, root.p, ecc.p);
            k_deepest<<<GV, kTB, 0, st>>>(vis.p, nvis, level.p, root.p, ecc.p, ip, best.p);
            k_reset_level<<<GV, kTB, 0, st>>>(vis.p, nvis, level.p);
            RC(cudaMemsetAsync(d_cnt.p, 0, sizeof(int), st));
            k_walk<<<GC, kTB, 0, st>>>(comps.p, ncomp, cand_x.p, ecc_x.p, cand_y.p, ecc.p, best.p, active.p,
                                       d_cnt.p, first);
            RC(cudaGetLastError());
            int nactive = 0;
            if (int rc = read_int(d_cnt.p, &nactive, st)) return rc;
            if (nactive == 0) break;
        }
        // 5. Cuthill-McKee levels, all components in lockstep
        RC(cudaMemsetAsync(parent.p, 0xff, sizeof(unsigned long long) * n, st));
        k_cm_start<<<GC, kTB, 0, st>>>(comps.p, ncomp, cand_x.p, base.p, pos.p, next_free.p, vis.p);
        RC(cudaGetLastError());
        const int nbits = bits_for(n);
        int64_t a = 0, b = ncomp;
        while (b > a) {
            RC(cudaMemsetAsync(d_cnt.p, 0, sizeof(int), st));
            k_expand_cm<<<blocks_for(b - a), kTB, 0, st>>>(vis.p + a, (int)(b - a), ip, ix, pos.p, parent.p,
                                                            vis.p + b, d_cnt.p);
            RC(cudaGetLastError());
            int fn = 0;
            if (int rc = read_int(d_cnt.p, &fn, st)) return rc;
            if (fn == 0) break;
            int32_t *lvl = vis.p + b;
            size_t t1 = tb;
            RC(cub::DeviceRadixSort::SortKeys(temp.p, t1, lvl, tmp.p, fn, 0, nbits, st));
            k_cm_key<<<blocks_for(fn), kTB, 0, st>>>(tmp.p, fn, parent.p, ip, key.p);
            size_t t2 = tb;
            RC(cub::DeviceRadixSort::SortPairs(temp.p, t2, key.p, key_alt.p, tmp.p, lvl, fn, 0, 64, st));
            k_place<<<blocks_for(fn), kTB, 0, st>>>(lvl, fn, root.p, pos.p, next_free.p);
            k_advance<<<blocks_for(fn), kTB, 0, st>>>(lvl, fn, root.p, next_free.p);
            RC(cudaGetLastError());
            a = b;
            b += fn;
        }
    }
    // 6. reverse
    k_forward<<<G, kTB, 0, st>>>(n, pos.p, forward);
    RC(cudaGetLastError());
    RC(cudaStreamSynchronize(st));
    return PARS3_OK;
}

}  // namespace

extern "C" int pars3_rcm_order_device(int64_t n, const int64_t *indptr, const int32_t *indices,
                                      int64_t *forward, void *stream) {
    if (n < 0 || n >= INT32_MAX || (n > 0 && (!indptr || !forward)))
        PARS3_FAIL(PARS3_ERR_ARG, "rcm_order_device: bad arguments");
    return rcm_device(n, indptr, indices, forward, (cudaStream_t)stream);
}

extern "C" int pars3_rcm_order_lower_device(int64_t n, const int64_t *row_ptr, const int32_t *col_ind,
                                            int64_t nnz, int64_t *forward, void *stream) {
    if (n < 0 || n >= INT32_MAX || nnz < 0 || (n > 0 && (!row_ptr || !forward)))
        PARS3_FAIL(PARS3_ERR_ARG, "rcm_order_lower_device: bad arguments");
    if (n == 0) return PARS3_OK;
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf<int64_t> cnt, ip;
    DevBuf<int32_t> ix;
    RC(cnt.alloc(n));
    RC(ip.alloc(n + 1));
    RC(ix.alloc(2 * nnz));
    RC(cudaMemsetAsync(cnt.p, 0, sizeof(int64_t) * n, st));
    const int G = blocks_for(n);
    k_deg_lower<<<G, kTB, 0, st>>>(n, row_ptr, col_ind, cnt.p);
    RC(cudaGetLastError());
    size_t tb = 0;
    RC(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, ip.p, n, st));
    DevBuf<uint8_t> temp;
    RC(temp.alloc(tb));
    RC(cub::DeviceScan::ExclusiveSum(temp.p, tb, cnt.p, ip.p, n, st));
    const int64_t total = 2 * nnz;
    RC(cudaMemcpyAsync(ip.p + n, &total, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    RC(cudaMemcpyAsync(cnt.p, ip.p, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st));  // fill cursors
    k_fill_lower<<<G, kTB, 0, st>>>(n, row_ptr, col_ind, cnt.p, ix.p);
    RC(cudaGetLastError());
    return rcm_device(n, ip.p, ix.p, forward, st);
}

// Internal (locality.cpp): RCM of a symmetric pattern held in HOST arrays,
// computed on the current device when there is one: upload, rcm_device, the
// labels back.  Returns non-zero (without setting an error the caller must
// report) when no device is usable; the caller then runs the host RCM, which
// gives the same labels bit for bit.
extern "C" int pars3_rcm_order_via_device(int64_t n, const int64_t *indptr, const int32_t *indices,
                                          int64_t *forward) {
    int dev = 0;
    if (n <= 0 || n >= INT32_MAX || cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return PARS3_ERR_CUDA;
    }
    const int64_t m2 = indptr[n];
    DevBuf<int64_t> ip, fw;
    DevBuf<int32_t> ix;
    if (ip.alloc(n + 1) != cudaSuccess || ix.alloc(m2) != cudaSuccess || fw.alloc(n) != cudaSuccess ||
        cudaMemcpy(ip.p, indptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice) != cudaSuccess ||
        (m2 > 0 && cudaMemcpy(ix.p, indices, sizeof(int32_t) * m2, cudaMemcpyHostToDevice) != cudaSuccess)) {
        cudaGetLastError();
        return PARS3_ERR_CUDA;
    }
    const int rc = rcm_device(n, ip.p, ix.p, fw.p, nullptr);
    if (rc) return rc;
    if (cudaMemcpy(forward, fw.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        return PARS3_ERR_CUDA;
    }
    return PARS3_OK;
}
