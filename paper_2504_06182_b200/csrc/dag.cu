// Occupancy dependency DAG over one-bend grid paths (sm_100a).
//
// Reference: occupancy_dag, /root/reference/proj/src/virtual_line.cpp:241-268.
// Edge (s, i) when path i visits source(s); edge (i, t) when path i visits
// target(t); s != i, t != i; the edge set is deduplicated and sorted by (a, b).
//
// Device form: two grid-sized lookup planes (source_of, target_of), one
// thread per path walking its staircase (horizontal along the source row,
// then vertical, virtual_line.cpp:150-173).  The only duplicate pair is an
// edge produced by both rules, i.e. (a, b) with b visiting source(a) AND a
// visiting target(b); rule 2 drops it when rule 1 already emits it, tested in
// O(1) against b's staircase.  Edges are packed as (a << 32 | b) and radix
// sorted, which yields the reference's lexicographic order.

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "dag.cuh"

namespace rb {

__device__ __forceinline__ bool on_path(int H, int32_t s, int32_t t, int32_t v) {
    const int xs = s / H, ys = s % H, xt = t / H, yt = t % H, x = v / H, y = v % H;
    if (y == ys && x >= min(xs, xt) && x <= max(xs, xt)) return true;      // horizontal leg
    if (x == xt && y >= min(ys, yt) && y <= max(ys, yt)) return true;      // vertical leg
    return false;
}

__global__ void dag_mark_kernel(int P, const int32_t *src, const int32_t *dst, int32_t *source_of,
                                int32_t *target_of) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
        source_of[src[i]] = i;
        target_of[dst[i]] = i;
    }
}

// pass 0 counts edges per path into cnt[i]; pass 1 writes them at off[i]
template <bool WRITE>
__global__ void dag_walk_kernel(int H, int P, const int32_t *src, const int32_t *dst, const int32_t *source_of,
                                const int32_t *target_of, int32_t *cnt, const int64_t *off,
                                unsigned long long *keys) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
        const int32_t s = src[i], t = dst[i];
        const int xs = s / H, ys = s % H, xt = t / H, yt = t % H;
        int n = 0;
        int64_t o = WRITE ? off[i] : 0;
        const int dx = xt > xs ? 1 : -1, dy = yt > ys ? 1 : -1;
        int x = xs, y = ys;
        for (;;) {
            const int32_t v = x * H + y;
            const int32_t a = source_of[v];
            if (a >= 0 && a != i) {
                if (WRITE) keys[o++] = ((unsigned long long)(uint32_t)a << 32) | (uint32_t)i;
                ++n;
            }
            const int32_t b = target_of[v];
            if (b >= 0 && b != i && !on_path(H, src[b], dst[b], s)) {
                if (WRITE) keys[o++] = ((unsigned long long)(uint32_t)i << 32) | (uint32_t)b;
                ++n;
            }
            if (x != xt) x += dx;
            else if (y != yt) y += dy;
            else break;
        }
        if (!WRITE) cnt[i] = n;
    }
}

__global__ void dag_unpack_kernel(int64_t n, const unsigned long long *keys, int32_t *a, int32_t *b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        a[i] = (int32_t)(keys[i] >> 32);
        b[i] = (int32_t)(keys[i] & 0xffffffffull);
    }
}

__global__ void widen_kernel(int n, const int32_t *in, int64_t *out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[i];
}

size_t dag_temp_bytes(int64_t max_edges, int P) {
    size_t t1 = 0, t2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, t1, (unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                   (int)max_edges);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, (int64_t *)nullptr, (int64_t *)nullptr, P + 1);
    return t1 > t2 ? t1 : t2;
}

cudaError_t dag_count(const DagArgs &d, cudaStream_t st, int64_t *n_edges_host) {
    const int threads = 256;
    cudaMemsetAsync(d.source_of, 0xff, (size_t)d.W * d.H * 4, st);
    cudaMemsetAsync(d.target_of, 0xff, (size_t)d.W * d.H * 4, st);
    const int blocks = (int)std::min<int64_t>((d.P + threads - 1) / threads + 1, 148 * 16);
    dag_mark_kernel<<<blocks, threads, 0, st>>>(d.P, d.src, d.dst, d.source_of, d.target_of);
    dag_walk_kernel<false><<<blocks, threads, 0, st>>>(d.H, d.P, d.src, d.dst, d.source_of, d.target_of, d.cnt,
                                                        nullptr, nullptr);
    widen_kernel<<<blocks, threads, 0, st>>>(d.P, d.cnt, d.off);
    cudaMemsetAsync(d.off + d.P, 0, 8, st);
    size_t tb = d.temp_bytes;
    cub::DeviceScan::ExclusiveSum(d.temp, tb, d.off, d.off, d.P + 1, st);
    cudaError_t e = cudaMemcpyAsync(n_edges_host, d.off + d.P, 8, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t dag_emit(const DagArgs &d, int64_t n_edges, cudaStream_t st, int32_t *ea, int32_t *eb) {
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((d.P + threads - 1) / threads + 1, 148 * 16);
    dag_walk_kernel<true><<<blocks, threads, 0, st>>>(d.H, d.P, d.src, d.dst, d.source_of, d.target_of, nullptr,
                                                       d.off, d.keys);
    size_t tb = d.temp_bytes;
    cub::DeviceRadixSort::SortKeys(d.temp, tb, d.keys, d.keys_alt, (int)n_edges, 0, 64, st);
    const int eblocks = (int)std::min<int64_t>((n_edges + threads - 1) / threads + 1, 148 * 16);
    dag_unpack_kernel<<<eblocks, threads, 0, st>>>(n_edges, d.keys_alt, ea, eb);
    return cudaGetLastError();
}

}  // namespace rb

// --------------------------------------------------------------------------
// occupancy_dag over explicit vertex lists (any path shape, e.g. aro's):
// every candidate pair is emitted, then sorted and deduplicated
// (virtual_line.cpp:261-262).
// --------------------------------------------------------------------------

namespace rb {

__global__ void dagx_mark_kernel(int P, const int64_t *off, const int32_t *verts, int32_t *source_of,
                                 int32_t *target_of) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
        source_of[verts[off[i]]] = i;
        target_of[verts[off[i + 1] - 1]] = i;
    }
}

template <bool WRITE>
__global__ void dagx_walk_kernel(int P, const int64_t *off, const int32_t *verts, const int32_t *source_of,
                                 const int32_t *target_of, int32_t *cnt, const int64_t *eoff,
                                 unsigned long long *keys) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
        int n = 0;
        int64_t o = WRITE ? eoff[i] : 0;
        for (int64_t q = off[i]; q < off[i + 1]; ++q) {
            const int32_t v = verts[q];
            const int32_t a = source_of[v];
            if (a >= 0 && a != i) {
                if (WRITE) keys[o++] = ((unsigned long long)(uint32_t)a << 32) | (uint32_t)i;
                ++n;
            }
            const int32_t b = target_of[v];
            if (b >= 0 && b != i) {
                if (WRITE) keys[o++] = ((unsigned long long)(uint32_t)i << 32) | (uint32_t)b;
                ++n;
            }
        }
        if (!WRITE) cnt[i] = n;
    }
}

__global__ void unique_flags_kernel(int64_t n, const unsigned long long *k, int32_t *flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

__global__ void unique_scatter_kernel(int64_t n, const unsigned long long *k, const int32_t *flag,
                                      const int64_t *pos, int32_t *a, int32_t *b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (flag[i]) {
            a[pos[i]] = (int32_t)(k[i] >> 32);
            b[pos[i]] = (int32_t)(k[i] & 0xffffffffull);
        }
}

}  // namespace rb

namespace rb {
template __global__ void dagx_walk_kernel<false>(int, const int64_t *, const int32_t *, const int32_t *,
                                                 const int32_t *, int32_t *, const int64_t *, unsigned long long *);
template __global__ void dagx_walk_kernel<true>(int, const int64_t *, const int32_t *, const int32_t *,
                                                const int32_t *, int32_t *, const int64_t *, unsigned long long *);
}  // namespace rb
