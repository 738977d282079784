// Wire formats: the reference's solution and batch
// schedule JSON (io.hpp:21-27, io.cpp:81-164), byte for byte, written on the
// device from the solver's own buffers.
//
// The reference prints through nlohmann::ordered_json::dump(2) (its vendor/
// json.hpp is not in the reference tree).  This restates the stock library's
// layout: objects and arrays open on their own line, one value per line, two
// spaces per level, ", " never used, "[]" for an empty array, keys in
// insertion order, and a trailing newline added by io.cpp.
//
// Every array element (a move, a dag edge, a path vertex, a batched move) is
// one text item; its bytes depend only on its own numbers and on whether it
// opens or closes its enclosing array.  So one kernel measures every item,
// a scan gives the offsets and a second kernel writes the items in place.
// The same device function does both (Writer<false> counts, Writer<true>
// writes), so lengths and bytes cannot drift apart.

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <string>
#include <vector>

#include "capi_internal.cuh"

using namespace rb;

namespace {

#define CK(call, where)                                             \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return cuda_fail(e_, where, detail); \
    } while (0)

template <bool WRITE>
struct Writer {
    char *p;
    int64_t n = 0;
    __host__ __device__ void put(char c) {
        if (WRITE) p[n] = c;
        ++n;
    }
    __host__ __device__ void str(const char *s) {
        while (*s) put(*s++);
    }
    __host__ __device__ void sp(int k) {
        for (int i = 0; i < k; ++i) put(' ');
    }
    __host__ __device__ void num(long long v) {
        if (v < 0) {
            put('-');
            v = -v;
        }
        char d[20];
        int k = 0;
        do {
            d[k++] = (char)('0' + v % 10);
            v /= 10;
        } while (v);
        while (k) put(d[--k]);
    }
    // [x, y] at indent `ind` (the caller wrote the leading indent)
    __host__ __device__ void xy(int ind, int x, int y) {
        str("[\n");
        sp(ind + 2);
        num(x);
        str(",\n");
        sp(ind + 2);
        num(y);
        put('\n');
        sp(ind);
        put(']');
    }
    // [[x1, y1], [x2, y2]] at indent `ind`, leading indent included
    __host__ __device__ void move(int ind, int H, int from, int to) {
        sp(ind);
        str("[\n");
        sp(ind + 2);
        xy(ind + 2, from / H, from % H);
        str(",\n");
        sp(ind + 2);
        xy(ind + 2, to / H, to % H);
        put('\n');
        sp(ind);
        put(']');
    }
};

// one-bend path (virtual_line.cpp:150-173): vertex k of s -> t
__host__ __device__ __forceinline__ int path_vertex(int H, int s, int t, int k) {
    const int xs = s / H, ys = s % H, xt = t / H, yt = t % H;
    const int nh = xt > xs ? xt - xs : xs - xt;
    if (k <= nh) return (xs + (xt > xs ? k : -k)) * H + ys;
    const int d = k - nh;
    return xt * H + ys + (yt > ys ? d : -d);
}
__host__ __device__ __forceinline__ int path_len(int H, int s, int t) {
    const int dx = s / H - t / H, dy = s % H - t % H;
    return (dx < 0 ? -dx : dx) + (dy < 0 ? -dy : dy);
}

struct Paths {
    int H, P;
    const int32_t *src, *dst, *order;  // order: schedule order of the paths (null = identity)
    const int64_t *moff;               // [P + 1] move offsets in schedule order
    const int64_t *voff;               // [P + 1] vertex offsets in path order
};

__device__ __forceinline__ int upper(const int64_t *off, int n, int64_t x) {  // last i with off[i] <= x
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= x) lo = mid;
        else hi = mid;
    }
    return lo;
}

// section items ---------------------------------------------------------------

template <bool W>
__device__ void item_move(Writer<W> &w, const Paths &ps, int64_t e) {  // "moves"[e], indent 4
    const int i = upper(ps.moff, ps.P, e);
    const int q = ps.order ? ps.order[i] : i;
    const int k = (int)(e - ps.moff[i]);
    if (e > 0) w.str(",\n");
    w.move(4, ps.H, path_vertex(ps.H, ps.src[q], ps.dst[q], k), path_vertex(ps.H, ps.src[q], ps.dst[q], k + 1));
}

template <bool W>
__device__ void item_edge(Writer<W> &w, const int32_t *a, const int32_t *b, int64_t e) {  // "dag_edges"[e]
    if (e > 0) w.str(",\n");
    w.sp(4);
    w.str("[\n");
    w.sp(6);
    w.num(a[e]);
    w.str(",\n");
    w.sp(6);
    w.num(b[e]);
    w.put('\n');
    w.sp(4);
    w.put(']');
}

template <bool W>
__device__ void item_vertex(Writer<W> &w, const Paths &ps, int64_t e) {  // vertex e of "paths"
    const int q = upper(ps.voff, ps.P, e);
    const int k = (int)(e - ps.voff[q]);
    const bool last = e + 1 == ps.voff[q + 1];
    if (k == 0) {
        if (q > 0) w.str(",\n");
        w.sp(4);
        w.str("[\n");
    } else {
        w.str(",\n");
    }
    const int v = path_vertex(ps.H, ps.src[q], ps.dst[q], k);
    w.sp(6);
    w.xy(6, v / ps.H, v % ps.H);
    if (last) {
        w.put('\n');
        w.sp(4);
        w.put(']');
    }
}

struct Batches {
    Paths ps;
    const int32_t *mb;       // batch per move (path-major)
    const uint32_t *sorted;  // move indices sorted by batch (stable: ascending path id)
    const uint32_t *skey;    // their batches
    int64_t D;
    int preset;
};

template <bool W>
__device__ void item_bmove(Writer<W> &w, const Batches &bs, int64_t e) {  // e-th move in batch order
    const int64_t m = bs.sorted[e];
    const int b = (int)bs.skey[e];
    const bool first = e == 0 || bs.skey[e - 1] != (uint32_t)b;
    const bool last = e + 1 == bs.D || bs.skey[e + 1] != (uint32_t)b;
    const int q = upper(bs.ps.moff, bs.ps.P, m);
    const int k = (int)(m - bs.ps.moff[q]);
    const int H = bs.ps.H;
    const int from = path_vertex(H, bs.ps.src[q], bs.ps.dst[q], k), to = path_vertex(H, bs.ps.src[q], bs.ps.dst[q], k + 1);
    if (first) {
        if (e > 0) w.str(",\n");
        w.sp(4);
        w.str("{\n");
        // tags from the batch's first move (batching.cpp:150-155; none -> null)
        const char *ax = "null", *dr = "null";
        if (bs.preset == RECON_PRESET_COLUMN_DIRECTION) {
            const int fx = from / H, fy = from % H, tx = to / H, ty = to % H;
            if (ty > fy) ax = "\"col\"", dr = "\"up\"";
            else if (ty < fy) ax = "\"col\"", dr = "\"down\"";
            else if (tx < fx) ax = "\"row\"", dr = "\"left\"";
            else ax = "\"row\"", dr = "\"right\"";
        }
        w.sp(6);
        w.str("\"axis\": ");
        w.str(ax);
        w.str(",\n");
        w.sp(6);
        w.str("\"dir\": ");
        w.str(dr);
        w.str(",\n");
        w.sp(6);
        w.str("\"moves\": [\n");
    } else {
        w.str(",\n");
    }
    w.move(8, H, from, to);
    if (last) {
        w.put('\n');
        w.sp(6);
        w.str("]\n");
        w.sp(4);
        w.put('}');
    }
}

// kernels ---------------------------------------------------------------------

enum Section { SEC_MOVES, SEC_EDGES, SEC_VERTICES, SEC_BMOVES };

struct Sec {
    Paths ps;
    Batches bs;
    const int32_t *ea, *eb;
};

template <bool W>
__device__ void item(int sec, const Sec &s, Writer<W> &w, int64_t e) {
    switch (sec) {
        case SEC_MOVES: item_move(w, s.ps, e); break;
        case SEC_EDGES: item_edge(w, s.ea, s.eb, e); break;
        case SEC_VERTICES: item_vertex(w, s.ps, e); break;
        default: item_bmove(w, s.bs, e); break;
    }
}

__global__ void k_measure(int sec, Sec s, int64_t n, int64_t *len) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        Writer<false> w{nullptr};
        item(sec, s, w, e);
        len[e] = w.n;
    }
}

// Writes 32 consecutive items per warp: each lane formats its item into the
// warp's shared-memory buffer (co-aligned with the destination), then the
// warp stores the group's bytes with 16-byte vector stores.  A group longer
// than the buffer is written item by item.
constexpr int kWriteWarps = 8, kWarpBuf = 8192;

__global__ void __launch_bounds__(kWriteWarps * 32) k_write(int sec, Sec s, int64_t n, const int64_t *off, char *out) {
    extern __shared__ __align__(16) char wbuf[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char *buf = wbuf + (size_t)warp * (kWarpBuf + 16);
    const int64_t ngroups = (n + 31) / 32;
    for (int64_t g = (int64_t)blockIdx.x * kWriteWarps + warp; g < ngroups; g += (int64_t)gridDim.x * kWriteWarps) {
        const int64_t e0 = g * 32, e1 = min(n, e0 + 32), e = e0 + lane;
        const int64_t base = off[e0], tot = off[e1] - base;
        char *dst = out + base;
        if (tot > kWarpBuf) {
            if (e < e1) {
                Writer<true> w{out + off[e]};
                item(sec, s, w, e);
            }
            continue;
        }
        const int mis = (int)((uintptr_t)dst & 15);
        char *b = buf + mis;  // b[i] goes to dst[i]; buf + 16 and dst + (16 - mis) share alignment
        if (e < e1) {
            Writer<true> w{b + (off[e] - base)};
            item(sec, s, w, e);
        }
        __syncwarp();
        const int head = (int)min(tot, (int64_t)((16 - mis) & 15));
        if (lane < head) dst[lane] = b[lane];
        const int64_t nvec = (tot - head) / 16;
        const uint4 *src4 = (const uint4 *)(b + head);
        uint4 *dst4 = (uint4 *)(dst + head);
        for (int64_t j = lane; j < nvec; j += 32) dst4[j] = src4[j];
        for (int64_t i = head + nvec * 16 + lane; i < tot; i += 32) dst[i] = b[i];
        __syncwarp();
    }
}

__global__ void k_path_lens(int H, int P, const int32_t *src, const int32_t *dst, const int32_t *order,
                            int64_t *moff, int64_t *voff) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
        const int q = order ? order[i] : i;
        moff[i] = path_len(H, src[q], dst[q]);
        voff[i] = path_len(H, src[i], dst[i]) + 1;
    }
}

__global__ void k_batch_keys(int64_t D, const int32_t *mb, uint32_t *key, uint32_t *idx) {
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < D; m += (int64_t)gridDim.x * blockDim.x) {
        key[m] = (uint32_t)mb[m];
        idx[m] = (uint32_t)m;
    }
}

int blocks_for(int64_t n, int sms) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8));
}

// host-side fixed text --------------------------------------------------------

std::string stats_tail(long long displaced, long long total) {
    return "  \"stats\": {\n    \"displaced_tokens\": " + std::to_string(displaced) +
           ",\n    \"total_displacement\": " + std::to_string(total) + "\n  }\n}\n";
}

struct Piece {  // fixed text or a device section
    std::string text;
    int sec = -1;
    int64_t n = 0;
};

// lays out the pieces, measures the sections, writes everything to out
recon_status assemble(Ctx *c, const std::vector<Piece> &pieces, const Sec &s, char *out, int64_t capacity,
                      int64_t *length, bool host) {
    int32_t *detail = nullptr;
    // every section gets its own (n + 1)-entry segment of item lengths -> offsets
    std::vector<int64_t> seg(pieces.size() + 1, 0), bytes(pieces.size(), 0);
    for (size_t i = 0; i < pieces.size(); ++i) seg[i + 1] = seg[i] + (pieces[i].sec >= 0 ? pieces[i].n + 1 : 0);
    int64_t *len = c->dev<int64_t>(S_W_LEN, (size_t)seg.back() + 1);
    if (!len) return cuda_fail(cudaErrorMemoryAllocation, "json workspace", detail);
    for (size_t i = 0; i < pieces.size(); ++i) {
        const Piece &p = pieces[i];
        if (p.sec < 0) {
            bytes[i] = (int64_t)p.text.size();
            continue;
        }
        int64_t *l = len + seg[i];
        CK(cudaMemsetAsync(l + p.n, 0, 8, c->stream), "memset");
        if (p.n) k_measure<<<blocks_for(p.n, c->sms), 256, 0, c->stream>>>(p.sec, s, p.n, l);
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, l, l, p.n + 1, c->stream);
        void *temp = c->get(S_TEMP, tb);
        if (!temp) return cuda_fail(cudaErrorMemoryAllocation, "json scan", detail);
        CK(cub::DeviceScan::ExclusiveSum(temp, tb, l, l, p.n + 1, c->stream), "scan");
        CK(cudaMemcpyAsync(&bytes[i], l + p.n, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
        c->launches += 2;
    }
    CK(cudaStreamSynchronize(c->stream), "D2H");
    std::vector<int64_t> start(pieces.size() + 1, 0);
    for (size_t i = 0; i < pieces.size(); ++i) start[i + 1] = start[i] + bytes[i];
    *length = start.back();
    if (capacity < *length) return RECON_ERR_CAPACITY;
    char *dout = host ? c->dev<char>(S_W_OUT, (size_t)*length + 1) : out;
    if (!dout) return cuda_fail(cudaErrorMemoryAllocation, "json output", detail);
    for (size_t i = 0; i < pieces.size(); ++i) {
        const Piece &p = pieces[i];
        if (p.sec < 0) {
            if (!p.text.empty()) {
                CK(cudaMemcpyAsync(dout + start[i], p.text.data(), p.text.size(), cudaMemcpyHostToDevice, c->stream),
                   "H2D");
                CK(cudaStreamSynchronize(c->stream), "H2D");  // pageable source
            }
            continue;
        }
        if (!p.n) continue;
        const int smem = kWriteWarps * (kWarpBuf + 16);
        CK(cudaFuncSetAttribute(k_write, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
        const int64_t groups = (p.n + 31) / 32;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((groups + kWriteWarps - 1) / kWriteWarps,
                                                                       (int64_t)c->sms * 3));
        k_write<<<grid, kWriteWarps * 32, smem, c->stream>>>(p.sec, s, p.n, len + seg[i], dout + start[i]);
        c->launches += 1;
    }
    CK(cudaGetLastError(), "json kernels");
    if (host) CK(cudaMemcpyAsync(out, dout, (size_t)*length, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaStreamSynchronize(c->stream), "json");
    return RECON_OK;
}

template <class T>
const T *stage(Ctx *c, int slot, const T *p, size_t n, bool host) {
    if (!host || !p) return p;
    T *d = c->dev<T>(slot, n ? n : 1);
    if (d && n) cudaMemcpyAsync(d, p, n * sizeof(T), cudaMemcpyHostToDevice, c->stream);
    return d;
}

// path offsets (schedule order for moves, path order for vertices); returns D
recon_status path_offsets(Ctx *c, Paths &ps, int64_t *D, int64_t *V) {
    int32_t *detail = nullptr;
    int64_t *moff = c->dev<int64_t>(S_W_MOFF, (size_t)ps.P + 1), *voff = c->dev<int64_t>(S_W_VOFF, (size_t)ps.P + 1);
    if (!moff || !voff) return cuda_fail(cudaErrorMemoryAllocation, "json paths", detail);
    CK(cudaMemsetAsync(moff + ps.P, 0, 8, c->stream), "memset");
    CK(cudaMemsetAsync(voff + ps.P, 0, 8, c->stream), "memset");
    if (ps.P) k_path_lens<<<blocks_for(ps.P, c->sms), 256, 0, c->stream>>>(ps.H, ps.P, ps.src, ps.dst, ps.order, moff, voff);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, moff, moff, ps.P + 1, c->stream);
    void *temp = c->get(S_TEMP, tb);
    if (!temp) return cuda_fail(cudaErrorMemoryAllocation, "json scan", detail);
    CK(cub::DeviceScan::ExclusiveSum(temp, tb, moff, moff, ps.P + 1, c->stream), "scan");
    CK(cub::DeviceScan::ExclusiveSum(temp, tb, voff, voff, ps.P + 1, c->stream), "scan");
    CK(cudaMemcpyAsync(D, moff + ps.P, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaMemcpyAsync(V, voff + ps.P, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    CK(cudaStreamSynchronize(c->stream), "D2H");
    c->launches += 3;
    ps.moff = moff;
    ps.voff = voff;
    return RECON_OK;
}

recon_status solution_json(recon_ctx *ctx, int32_t width, int32_t height, int32_t path_count, const int32_t *path_src,
                           const int32_t *path_dst, const int32_t *path_order, int64_t dag_count, const int32_t *dag_a,
                           const int32_t *dag_b, int64_t displaced, int64_t total, char *out, int64_t capacity,
                           int64_t *length, bool host) {
    int32_t *detail = nullptr;
    if (!length || width <= 0 || height <= 0 || path_count < 0 || dag_count < 0) return RECON_ERR_ARGUMENT;
    if ((path_count && (!path_src || !path_dst)) || (dag_count && (!dag_a || !dag_b))) return RECON_ERR_ARGUMENT;
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    Sec s{};
    s.ps.H = height;
    s.ps.P = path_count;
    s.ps.src = stage(c, S_PSRC, path_src, (size_t)path_count, host);
    s.ps.dst = stage(c, S_PDST, path_dst, (size_t)path_count, host);
    s.ps.order = stage(c, S_PEV, path_order, (size_t)path_count, host);
    s.ea = stage(c, S_EA, dag_a, (size_t)dag_count, host);
    s.eb = stage(c, S_EB, dag_b, (size_t)dag_count, host);
    int64_t D = 0, V = 0;
    recon_status st = path_offsets(c, s.ps, &D, &V);
    if (st != RECON_OK) return st;
    std::vector<Piece> pc;
    auto text = [&](std::string t) {
        Piece p;
        p.text = std::move(t);
        pc.push_back(std::move(p));
    };
    auto sec = [&](int k, int64_t n) {
        Piece p;
        p.sec = k;
        p.n = n;
        pc.push_back(std::move(p));
    };
    auto array = [&](const char *key, int k, int64_t n, bool comma) {
        if (!n) {
            text(std::string("  \"") + key + "\": []" + (comma ? ",\n" : "\n"));
            return;
        }
        text(std::string("  \"") + key + "\": [\n");
        sec(k, n);
        text(std::string("\n  ]") + (comma ? ",\n" : "\n"));
    };
    text("{\n");
    array("moves", SEC_MOVES, D, true);
    array("dag_edges", SEC_EDGES, dag_count, true);
    array("paths", SEC_VERTICES, path_count ? V : 0, true);
    text(stats_tail(displaced, total));
    return assemble(c, pc, s, out, capacity, length, host);
}

recon_status batch_json(recon_ctx *ctx, int32_t width, int32_t height, int32_t path_count, const int32_t *path_src,
                        const int32_t *path_dst, const int32_t *move_batch, int32_t batch_count, int32_t preset,
                        char *out, int64_t capacity, int64_t *length, bool host) {
    int32_t *detail = nullptr;
    if (!length || width <= 0 || height <= 0 || path_count < 0 || batch_count < 0) return RECON_ERR_ARGUMENT;
    if (path_count && (!path_src || !path_dst)) return RECON_ERR_ARGUMENT;
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    Sec s{};
    s.ps.H = height;
    s.ps.P = path_count;
    s.ps.src = stage(c, S_PSRC, path_src, (size_t)path_count, host);
    s.ps.dst = stage(c, S_PDST, path_dst, (size_t)path_count, host);
    s.ps.order = nullptr;
    int64_t D = 0, V = 0;
    recon_status st = path_offsets(c, s.ps, &D, &V);
    if (st != RECON_OK) return st;
    if (D && !move_batch) return RECON_ERR_ARGUMENT;
    s.bs.ps = s.ps;
    s.bs.mb = stage(c, S_W_MB, move_batch, (size_t)D, host);
    s.bs.D = D;
    s.bs.preset = preset;
    if (D) {  // batch-major order, stable in move index (= ascending path id within a batch)
        uint32_t *key = c->dev<uint32_t>(S_W_K0, (size_t)D), *key2 = c->dev<uint32_t>(S_W_K1, (size_t)D);
        uint32_t *idx = c->dev<uint32_t>(S_W_I0, (size_t)D), *idx2 = c->dev<uint32_t>(S_W_I1, (size_t)D);
        if (!key || !key2 || !idx || !idx2) return cuda_fail(cudaErrorMemoryAllocation, "json batches", detail);
        k_batch_keys<<<blocks_for(D, c->sms), 256, 0, c->stream>>>(D, s.bs.mb, key, idx);
        int bits = 1;
        while ((1ll << bits) < (int64_t)batch_count + 1 && bits < 32) ++bits;
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, idx, idx2, (int)D, 0, bits, c->stream);
        void *temp = c->get(S_TEMP, tb);
        if (!temp) return cuda_fail(cudaErrorMemoryAllocation, "json sort", detail);
        CK(cub::DeviceRadixSort::SortPairs(temp, tb, key, key2, idx, idx2, (int)D, 0, bits, c->stream), "sort");
        s.bs.sorted = idx2;
        s.bs.skey = key2;
        c->launches += 2;
    }
    std::vector<Piece> pc;
    Piece p;
    if (!D) {
        p.text = "{\n  \"batches\": []\n}\n";
        pc.push_back(p);
    } else {
        p.text = "{\n  \"batches\": [\n";
        pc.push_back(p);
        Piece q;
        q.sec = SEC_BMOVES;
        q.n = D;
        pc.push_back(q);
        Piece r;
        r.text = "\n  ]\n}\n";
        pc.push_back(r);
    }
    return assemble(c, pc, s, out, capacity, length, host);
}

}  // namespace

extern "C" {

recon_status recon_solution_json(recon_ctx *ctx, int32_t width, int32_t height, int32_t path_count,
                                 const int32_t *path_src, const int32_t *path_dst, const int32_t *path_order,
                                 int64_t dag_count, const int32_t *dag_a, const int32_t *dag_b,
                                 int64_t displaced_tokens, int64_t total_displacement, char *out, int64_t capacity,
                                 int64_t *length) {
    return solution_json(ctx, width, height, path_count, path_src, path_dst, path_order, dag_count, dag_a, dag_b,
                         displaced_tokens, total_displacement, out, capacity, length, false);
}

recon_status recon_solution_json_host(recon_ctx *ctx, int32_t width, int32_t height, int32_t path_count,
                                      const int32_t *path_src, const int32_t *path_dst, const int32_t *path_order,
                                      int64_t dag_count, const int32_t *dag_a, const int32_t *dag_b,
                                      int64_t displaced_tokens, int64_t total_displacement, char *out,
                                      int64_t capacity, int64_t *length) {
    return solution_json(ctx, width, height, path_count, path_src, path_dst, path_order, dag_count, dag_a, dag_b,
                         displaced_tokens, total_displacement, out, capacity, length, true);
}

recon_status recon_batch_schedule_json(recon_ctx *ctx, int32_t width, int32_t height, int32_t path_count,
                                       const int32_t *path_src, const int32_t *path_dst, const int32_t *move_batch,
                                       int32_t batch_count, int32_t preset, char *out, int64_t capacity,
                                       int64_t *length) {
    return batch_json(ctx, width, height, path_count, path_src, path_dst, move_batch, batch_count, preset, out,
                      capacity, length, false);
}

recon_status recon_batch_schedule_json_host(recon_ctx *ctx, int32_t width, int32_t height, int32_t path_count,
                                            const int32_t *path_src, const int32_t *path_dst,
                                            const int32_t *move_batch, int32_t batch_count, int32_t preset,
                                            char *out, int64_t capacity, int64_t *length) {
    return batch_json(ctx, width, height, path_count, path_src, path_dst, move_batch, batch_count, preset, out,
                      capacity, length, true);
}

}  // extern "C"
