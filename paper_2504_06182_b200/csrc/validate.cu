// On-device validators for grid solutions: batched
// restatements of the reference's
//   validate_solution        executor.cpp:142-183
//   check_one_move_per_token executor.cpp:185-219
//   validate_batches         batching.cpp:161-252
// for this ABI's path format (one-bend paths from (src, dst); the identity
// schedule = paths in order, each path's moves in order; batch index per move,
// path-major).
//
// The reference replays moves one by one.  Here every check is a parallel
// predicate over paths, moves or vertices:
//   - execution: before path i runs, vertex v holds a token iff
//       init(v) - [src_of(v) < i] + [dst_of(v) < i]
//     (sources and targets are distinct once the shared-vertex checks pass),
//     so a path is collision-free iff its source holds a token and every other
//     vertex on it is empty at that time; "some path collides" equals "the
//     sequential replay fails";
//   - one move per token: path i's first move takes the token that arrived
//     by the path ending at src_i, if that path ran earlier;
//   - batches: every move yields a departure and an arrival event keyed
//     (vertex, batch).  After a radix sort, a vertex's events must alternate
//     departure/arrival starting from its initial occupancy, and no key may
//     repeat (vertex-disjointness); per-batch counts and min/max of the
//     (direction, line) key give emptiness and the column_direction
//     constraint.
// Each report keeps the reference's check order and early returns, using the
// first failing path / batch index (atomicMin).  When a solution has shared
// endpoints or collisions, the one-move report follows the reference's
// match_schedule + token tracking exactly with a one-thread replay (on a
// collision-free schedule the match is the identity, so the parallel rule is
// exact).

#include <climits>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <vector>

#include "capi_internal.cuh"

using namespace rb;

namespace {

#define CK(call, where)                                             \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return cuda_fail(e_, where, detail); \
    } while (0)

// raw facts gathered by the kernels (atomicOr)
enum : unsigned {
    F_BOUNDS = 1u << 0,
    F_SHARED_S = 1u << 1,
    F_SHARED_T = 1u << 2,
    F_EXEC = 1u << 3,
    F_TARGETS = 1u << 4,
    F_EDGE_BACK = 1u << 5,   // some dag edge a >= b (a cycle is possible)
    F_DAG_ORDER = 1u << 6,   // some dag edge a > b between paths with moves
    F_BCONS = 1u << 7,
    F_BORDER = 1u << 8,
    F_BDAG = 1u << 9,
    F_BTARGETS = 1u << 10,
    F_CYCLE = 1u << 11,
    F_TOKMATCH = 1u << 12,
};

struct VState {
    unsigned raw;
    int moved;
    unsigned long long weight;
    int tok_empty, tok_second;                     // first path index
    int b_empty, b_constraint, b_disjoint, b_collision;  // first batch index
    int changed, alive;                            // cycle peeling
};

struct VArgs {
    int W, H, hp, wpc;
    const uint64_t *occ;
    const int32_t *src, *dst;
    int P;
    int32_t *src_of, *dst_of;  // [W*H] path index (max on duplicates, like the reference's maps)
    int64_t *len;              // [P + 1] -> exclusive scan = move offsets
    const int32_t *mb;         // batch per move or null
    int nb;
    int preset;
    unsigned long long *ev;    // [2 D] (vertex << 32 | batch << 1 | arrival)
    int32_t *bcnt, *bmin, *bmax;
    int8_t *fin;               // [W*H] occupancy after the last batch event, -1 = untouched
    VState *st;
};

__device__ __forceinline__ int init_occ(const VArgs &a, int v) {
    const int x = v / a.H, y = v % a.H;
    return (int)((a.occ[(size_t)x * a.wpc + (y >> 6)] >> (y & 63)) & 1ull);
}

__device__ __forceinline__ bool in_grid(const VArgs &a, int v) { return v >= 0 && v < a.W * a.H; }

// one-bend walk (virtual_line.cpp:150-173): k-th vertex of the path s -> t
struct Walk {
    int xs, ys, xt, yt, nh, n;
    __device__ Walk(int H, int s, int t) {
        xs = s / H;
        ys = s % H;
        xt = t / H;
        yt = t % H;
        nh = xt > xs ? xt - xs : xs - xt;
        n = nh + (yt > ys ? yt - ys : ys - yt);  // moves
    }
    __device__ __forceinline__ int at(int H, int k) const {
        if (k <= nh) return (xs + (xt > xs ? k : -k)) * H + ys;
        const int d = k - nh;
        return xt * H + ys + (yt > ys ? d : -d);
    }
};

__global__ void k_paths(VArgs a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.P; i += gridDim.x * blockDim.x) {
        const int s = a.src[i], t = a.dst[i];
        if (!in_grid(a, s) || !in_grid(a, t)) {  // check_paths: "leaves the grid"
            atomicOr(&a.st->raw, F_BOUNDS);
            a.len[i] = 0;
            continue;
        }
        const Walk w(a.H, s, t);
        a.len[i] = w.n;
        atomicAdd(&a.st->weight, (unsigned long long)w.n);
        if (w.n > 0) atomicAdd(&a.st->moved, 1);
        if (atomicMax(&a.src_of[s], i) >= 0) atomicOr(&a.st->raw, F_SHARED_S);
        if (atomicMax(&a.dst_of[t], i) >= 0) atomicOr(&a.st->raw, F_SHARED_T);
    }
}

__device__ __forceinline__ int first_batch(const VArgs &a, int p) {
    return a.len[p + 1] > a.len[p] ? a.mb[a.len[p]] : -1;  // len holds offsets after the scan
}

// per path: execution, one-move, implicit (occupancy) dag, batch events
template <bool IMPLICIT_DAG>
__global__ void k_walk(VArgs a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.P; i += gridDim.x * blockDim.x) {
        const int s = a.src[i], t = a.dst[i];
        if (!in_grid(a, s) || !in_grid(a, t)) continue;
        const Walk w(a.H, s, t);
        const int64_t off = a.len[i];
        auto occ_before = [&](int v) {
            const int sp = a.src_of[v], dp = a.dst_of[v];
            return init_occ(a, v) - (sp >= 0 && sp < i) + (dp >= 0 && dp < i);
        };
        unsigned raw = 0;
        // execution of the identity schedule (executor.cpp:10-26)
        if (w.n > 0) {
            const int o = occ_before(s);
            if (o != 1) raw |= F_EXEC;
            if (o <= 0) atomicMin(&a.st->tok_empty, i);
            const int dp = a.dst_of[s];
            if (o > 0 && dp >= 0 && dp < i) atomicMin(&a.st->tok_second, i);
        }
        const int fbi = a.mb && w.n > 0 ? a.mb[off] : -1;
        int prevb = -1;
        for (int k = 0; k <= w.n; ++k) {
            const int v = w.at(a.H, k);
            if (k > 0 && occ_before(v) != 0) raw |= F_EXEC;
            if (IMPLICIT_DAG) {  // occupancy_dag edges (virtual_line.cpp:241-268)
                const int sp = a.src_of[v], dp = a.dst_of[v];
                if (sp >= 0 && sp != i) {  // (sp, i)
                    if (sp > i) raw |= F_EDGE_BACK | (a.len[sp + 1] > a.len[sp] && w.n > 0 ? F_DAG_ORDER : 0u);
                    if (a.mb && w.n > 0) {
                        const int fb = first_batch(a, sp);
                        if (fb >= 0 && fbi < fb) raw |= F_BDAG;
                    }
                }
                if (dp >= 0 && dp != i) {  // (i, dp)
                    if (i > dp) raw |= F_EDGE_BACK | (a.len[dp + 1] > a.len[dp] && w.n > 0 ? F_DAG_ORDER : 0u);
                    if (a.mb && w.n > 0) {
                        const int fb = first_batch(a, dp);
                        if (fb >= 0 && fb < fbi) raw |= F_BDAG;
                    }
                }
            }
            if (a.mb && k < w.n) {  // move k: v -> next
                const int b = a.mb[off + k];
                unsigned long long *e = a.ev + 2 * (off + k);
                if (b < 0 || b >= a.nb) {
                    raw |= F_BCONS;
                    e[0] = e[1] = ~0ull;
                    continue;
                }
                if (b < prevb) raw |= F_BORDER;
                prevb = b;
                const int u = w.at(a.H, k + 1);
                e[0] = ((unsigned long long)v << 32) | ((unsigned long long)b << 1);
                e[1] = ((unsigned long long)u << 32) | ((unsigned long long)b << 1) | 1ull;
                atomicAdd(&a.bcnt[b], 1);
                if (a.preset == RECON_PRESET_COLUMN_DIRECTION) {  // move_dir / compatible (batching.cpp:9-24)
                    const int fx = v / a.H, fy = v % a.H, tx = u / a.H, ty = u % a.H;
                    const int dir = ty > fy ? 0 : ty < fy ? 1 : tx < fx ? 2 : 3;
                    const int key = (dir << 16) | (dir < 2 ? fx : fy);
                    atomicMin(&a.bmin[b], key);
                    atomicMax(&a.bmax[b], key);
                }
            }
        }
        if (raw) atomicOr(&a.st->raw, raw);
    }
}

// explicit dag edges: order, batch order, back edges
__global__ void k_edges(VArgs a, const int32_t *ea, const int32_t *eb, int64_t ne) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
        const int i = ea[e], j = eb[e];
        if (i < 0 || j < 0 || i >= a.P || j >= a.P) continue;
        const bool mi = a.len[i + 1] > a.len[i], mj = a.len[j + 1] > a.len[j];
        unsigned raw = 0;
        if (i >= j) raw |= F_EDGE_BACK;
        if (i > j && mi && mj) raw |= F_DAG_ORDER;
        if (a.mb && mi && mj && a.mb[a.len[j]] < a.mb[a.len[i]]) raw |= F_BDAG;
        if (raw) atomicOr(&a.st->raw, raw);
    }
}

// final configuration covers the band (canonical execution)
__global__ void k_targets(VArgs a) {
    const int ylo = (a.H - a.hp) / 2, n = a.W * a.hp;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        const int v = (c / a.hp) * a.H + ylo + c % a.hp;
        const int o = init_occ(a, v) - (a.src_of[v] >= 0) + (a.dst_of[v] >= 0);
        if (o != 1) atomicOr(&a.st->raw, F_TARGETS);
        if (a.mb) {
            const int f = a.fin[v] >= 0 ? a.fin[v] : init_occ(a, v);
            if (!f) atomicOr(&a.st->raw, F_BTARGETS);
        }
    }
}

// sorted batch events: disjointness, alternation, final occupancy
__global__ void k_events(VArgs a, const unsigned long long *ev, int64_t n) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long e = ev[k];
        if (e == ~0ull) continue;
        const int v = (int)(e >> 32), b = (int)((e >> 1) & 0x7fffffff), arr = (int)(e & 1);
        int before;
        if (k > 0 && (ev[k - 1] >> 32) == (unsigned long long)v) {
            const unsigned long long p = ev[k - 1];
            if ((int)((p >> 1) & 0x7fffffff) == b) atomicMin(&a.st->b_disjoint, b);
            before = (int)(p & 1);  // occupied after an arrival
        } else {
            before = init_occ(a, v);
        }
        if (arr ? before : !before) atomicMin(&a.st->b_collision, b);
        if (k + 1 == n || (ev[k + 1] >> 32) != (unsigned long long)v || ev[k + 1] == ~0ull) a.fin[v] = (int8_t)arr;
    }
}

__global__ void k_batches(VArgs a) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < a.nb; b += gridDim.x * blockDim.x) {
        if (a.bcnt[b] == 0) atomicMin(&a.st->b_empty, b);
        else if (a.preset == RECON_PRESET_COLUMN_DIRECTION && a.bmin[b] != a.bmax[b])
            atomicMin(&a.st->b_constraint, b);
    }
}

// cycle check by peeling sources (only when some edge points backwards)
__global__ void k_peel_mark(VArgs a, const int32_t *ea, const int32_t *eb, int64_t ne, const int8_t *alive,
                            int8_t *haspred) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
        const int i = ea[e], j = eb[e];
        if (i >= 0 && j >= 0 && i < a.P && j < a.P && alive[i] && alive[j]) haspred[j] = 1;
    }
}

__global__ void k_peel_remove(VArgs a, int8_t *alive, int8_t *haspred) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.P; i += gridDim.x * blockDim.x) {
        if (alive[i] && !haspred[i]) {
            alive[i] = 0;
            a.st->changed = 1;
        }
        if (alive[i]) a.st->alive = 1;
        haspred[i] = 0;
    }
}

// implicit dag edges, materialised for the cycle check
template <bool FILL>
__global__ void k_occ_edges(VArgs a, int64_t *cnt, int32_t *ea, int32_t *eb) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.P; i += gridDim.x * blockDim.x) {
        const int s = a.src[i], t = a.dst[i];
        int64_t n = 0, at = FILL ? cnt[i] : 0;
        if (in_grid(a, s) && in_grid(a, t)) {
            const Walk w(a.H, s, t);
            for (int k = 0; k <= w.n; ++k) {
                const int v = w.at(a.H, k), sp = a.src_of[v], dp = a.dst_of[v];
                if (sp >= 0 && sp != i) {
                    if (FILL) {
                        ea[at] = sp;
                        eb[at++] = i;
                    }
                    ++n;
                }
                if (dp >= 0 && dp != i) {
                    if (FILL) {
                        ea[at] = i;
                        eb[at++] = dp;
                    }
                    ++n;
                }
            }
        }
        if (!FILL) cnt[i] = n;
    }
}

// check_one_move_per_token exactly as the reference runs it, by one thread:
// match_schedule (executor.cpp:82-140) keeps each vertex's pending path fronts
// in insertion order and gives a move to the first pending path whose next
// vertex fits (on colliding schedules that can be another path than the one
// that produced the move); the token identities are followed alongside
// (executor.cpp:185-219).  buf: 3V + 3P ints.
__global__ void k_token_replay(VArgs a, int32_t *buf, int8_t *began) {
    if (blockIdx.x || threadIdx.x) return;
    const int V = a.W * a.H, P = a.P;
    int32_t *head = buf, *tail = buf + V, *tok = buf + 2 * V, *nx = buf + 3 * V, *pv = nx + P, *nk = pv + P;
    for (int v = 0; v < V; ++v) {
        head[v] = tail[v] = -1;
        tok[v] = init_occ(a, v) ? v : -1;
        began[v] = 0;
    }
    auto push = [&](int v, int q) {
        nx[q] = -1;
        pv[q] = tail[v];
        if (tail[v] >= 0) nx[tail[v]] = q;
        else head[v] = q;
        tail[v] = q;
    };
    for (int q = 0; q < P; ++q) {
        nk[q] = 0;
        if (a.len[q + 1] > a.len[q]) push(a.src[q], q);
    }
    int fail_tok = 0;  // first token failure (1 empty, 2 second path) while tracking
    for (int i = 0; i < P; ++i) {
        const Walk w(a.H, a.src[i], a.dst[i]);
        for (int k = 0; k < w.n; ++k) {
            const int from = w.at(a.H, k), to = w.at(a.H, k + 1);
            int m = -1;
            for (int q = head[from]; q >= 0; q = nx[q]) {
                const Walk wq(a.H, a.src[q], a.dst[q]);
                if (wq.at(a.H, nk[q] + 1) == to) {
                    m = q;
                    break;
                }
            }
            if (m < 0) {  // "scheduled move ... matches no pending path edge"
                a.st->tok_empty = a.st->tok_second = INT_MAX;
                a.st->raw |= F_TOKMATCH;
                return;
            }
            if (pv[m] >= 0) nx[pv[m]] = nx[m];
            else head[from] = nx[m];
            if (nx[m] >= 0) pv[nx[m]] = pv[m];
            else tail[from] = pv[m];
            const bool starts = nk[m] == 0;
            const int kk = ++nk[m];
            const Walk wm(a.H, a.src[m], a.dst[m]);
            if (kk < wm.n) push(wm.at(a.H, kk), m);
            if (!fail_tok) {
                const int tk = tok[from];
                if (tk < 0) {
                    fail_tok = 1;
                    a.st->tok_empty = i;
                } else if (starts && began[tk]) {
                    fail_tok = 2;
                    a.st->tok_second = i;
                } else {
                    if (starts) began[tk] = 1;
                    tok[from] = -1;
                    tok[to] = tk;
                }
            }
        }
    }
}

__global__ void k_init_state(VState *st) {
    st->raw = 0;
    st->moved = 0;
    st->weight = 0;
    st->tok_empty = st->tok_second = INT_MAX;
    st->b_empty = st->b_constraint = st->b_disjoint = st->b_collision = INT_MAX;
    st->changed = st->alive = 0;
}

__global__ void k_fill_i32(int32_t *p, int64_t n, int32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// the three reports, in the reference's order with its early returns
__global__ void k_verdict(VState *st, const int64_t *claim_td, const int32_t *claim_disp, int has_mb, int nb,
                          uint32_t *out) {
    if (blockIdx.x || threadIdx.x) return;
    const unsigned r = st->raw;
    uint32_t v = 0;
    if (r & F_BOUNDS) {  // a one-bend path needs in-grid endpoints; nothing else is evaluated
        *out = RECON_V_PATH_BOUNDS;
        return;
    }
    if (r & F_SHARED_S) v |= RECON_V_SHARED_SOURCE;
    if (r & F_SHARED_T) v |= RECON_V_SHARED_TARGET;
    if (r & F_CYCLE) v |= RECON_V_DAG_CYCLE;
    if (claim_td && (unsigned long long)*claim_td != st->weight) v |= RECON_V_STATS_DISPLACEMENT;
    if (claim_disp && *claim_disp != st->moved) v |= RECON_V_STATS_DISPLACED;
    if (!v) {  // validate_solution returns early on the checks above
        if (r & F_EXEC) {
            v |= RECON_V_EXECUTION;
        } else {
            if (r & F_TARGETS) v |= RECON_V_TARGETS;
            if (r & F_DAG_ORDER) v |= RECON_V_DAG_ORDER;
        }
    }
    if (r & F_TOKMATCH) v |= RECON_V_TOKEN_MATCH;
    else if (st->tok_empty != INT_MAX || st->tok_second != INT_MAX)
        v |= st->tok_empty <= st->tok_second ? RECON_V_TOKEN_EMPTY : RECON_V_TOKEN_SECOND_PATH;
    if (has_mb) {
        uint32_t bv = 0;
        if (r & F_BCONS) bv |= RECON_V_BATCH_CONSERVATION;
        if ((unsigned long long)nb > st->weight) bv |= RECON_V_BATCH_BOUND;
        const int bstar = min(st->b_disjoint, st->b_collision);
        if (st->b_empty < bstar) bv |= RECON_V_BATCH_EMPTY;
        if (st->b_constraint < bstar || (st->b_constraint == bstar && st->b_disjoint != bstar))
            bv |= RECON_V_BATCH_CONSTRAINT;
        if (bstar != INT_MAX) {
            bv |= st->b_disjoint == bstar ? RECON_V_BATCH_DISJOINT : RECON_V_BATCH_COLLISION;
        } else {
            if (r & F_BTARGETS) bv |= RECON_V_BATCH_TARGETS;
            if (!bv) {
                if (r & F_BORDER) bv |= RECON_V_BATCH_ORDER;
                else if (r & F_BDAG) bv |= RECON_V_BATCH_DAG;
            }
        }
        v |= bv;
    }
    *out = v;
}

int blocks_for(int64_t n, int sms) {
    const int64_t b = (n + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)sms * 8));
}

template <class T>
const T *stage_in(Ctx *c, int slot, const T *p, size_t n, bool host, cudaError_t *err) {
    if (!host || !p) return p;
    T *d = c->dev<T>(slot, n ? n : 1);
    if (!d) {
        *err = cudaErrorMemoryAllocation;
        return nullptr;
    }
    if (n) *err = cudaMemcpyAsync(d, p, n * sizeof(T), cudaMemcpyHostToDevice, c->stream);
    return d;
}

recon_status validate_impl(recon_ctx *ctx, const recon_validate_batch *b, bool host) {
    int32_t *detail = nullptr;
    if (!b || !b->occ || !b->path_src || !b->path_dst || !b->path_count || !b->verdict) return RECON_ERR_ARGUMENT;
    if (b->width <= 0 || b->height <= 0 || b->h_prime <= 0 || b->h_prime >= b->height) return RECON_ERR_ARGUMENT;
    if (b->dag_mode == RECON_DAG_EXPLICIT && (!b->dag_a || !b->dag_b || !b->dag_offset)) return RECON_ERR_ARGUMENT;
    if (b->move_batch && !b->batch_count) return RECON_ERR_ARGUMENT;
    if (b->count <= 0) return RECON_OK;
    Ctx *c = resolve(ctx);
    if (!c) return RECON_ERR_CUDA;
    CK(cudaSetDevice(c->device), "cudaSetDevice");
    const int n = b->count, W = b->width, H = b->height, wpc = (H + 63) / 64;
    const int64_t V = (int64_t)W * H;
    // per-instance sizes on the host
    std::vector<int32_t> pc(n), nbv(n, 0);
    std::vector<int64_t> eoff(n + 1, 0);
    if (host) {
        std::copy(b->path_count, b->path_count + n, pc.begin());
        if (b->batch_count) std::copy(b->batch_count, b->batch_count + n, nbv.begin());
        if (b->dag_mode == RECON_DAG_EXPLICIT) std::copy(b->dag_offset, b->dag_offset + n + 1, eoff.begin());
    } else {
        CK(cudaMemcpyAsync(pc.data(), b->path_count, n * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        if (b->batch_count)
            CK(cudaMemcpyAsync(nbv.data(), b->batch_count, n * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        if (b->dag_mode == RECON_DAG_EXPLICIT)
            CK(cudaMemcpyAsync(eoff.data(), b->dag_offset, (n + 1) * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
        CK(cudaStreamSynchronize(c->stream), "D2H");
    }
    uint32_t *d_verdict = host ? c->dev<uint32_t>(S_V_VERDICT, n) : b->verdict;
    VState *st = c->dev<VState>(S_V_STATE, 1);
    VArgs a{};
    a.W = W;
    a.H = H;
    a.hp = b->h_prime;
    a.wpc = wpc;
    a.preset = b->preset;
    a.src_of = c->dev<int32_t>(S_V_SRCOF, V);
    a.dst_of = c->dev<int32_t>(S_V_DSTOF, V);
    a.fin = c->dev<int8_t>(S_V_FIN, V);
    a.st = st;
    if (!d_verdict || !st || !a.src_of || !a.dst_of || !a.fin)
        return cuda_fail(cudaErrorMemoryAllocation, "validate workspace", detail);
    const int sms = c->sms;
    for (int i = 0; i < n; ++i) {
        cudaError_t err = cudaSuccess;
        const int P = pc[i];
        a.P = P;
        a.occ = stage_in(c, S_OCC, b->occ + (size_t)i * W * wpc, (size_t)W * wpc, host, &err);
        a.src = stage_in(c, S_PSRC, b->path_src + i * b->path_stride, (size_t)P, host, &err);
        a.dst = stage_in(c, S_PDST, b->path_dst + i * b->path_stride, (size_t)P, host, &err);
        const int64_t *ctd = b->total_displacement ? stage_in(c, S_TDISP, b->total_displacement + i, 1, host, &err) : nullptr;
        const int32_t *cdp = b->displaced ? stage_in(c, S_PCNT, b->displaced + i, 1, host, &err) : nullptr;
        if (err != cudaSuccess) return cuda_fail(err, "validate inputs", detail);
        a.len = c->dev<int64_t>(S_V_LEN, (size_t)P + 1);
        if (!a.len) return cuda_fail(cudaErrorMemoryAllocation, "validate workspace", detail);
        k_init_state<<<1, 1, 0, c->stream>>>(st);
        k_fill_i32<<<blocks_for(V, sms), 256, 0, c->stream>>>(a.src_of, V, -1);
        k_fill_i32<<<blocks_for(V, sms), 256, 0, c->stream>>>(a.dst_of, V, -1);
        CK(cudaMemsetAsync(a.fin, 0xff, (size_t)V, c->stream), "memset");
        CK(cudaMemsetAsync(a.len + P, 0, 8, c->stream), "memset");
        k_paths<<<blocks_for(P, sms), 256, 0, c->stream>>>(a);
        // move offsets
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, a.len, a.len, P + 1, c->stream);
        void *temp = c->get(S_TEMP, tb);
        if (!temp) return cuda_fail(cudaErrorMemoryAllocation, "validate scan", detail);
        CK(cub::DeviceScan::ExclusiveSum(temp, tb, a.len, a.len, P + 1, c->stream), "scan");
        int64_t D = 0;
        CK(cudaMemcpyAsync(&D, a.len + P, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
        CK(cudaStreamSynchronize(c->stream), "D2H");
        // batch inputs
        a.mb = nullptr;
        a.nb = nbv[i];
        if (b->move_batch) {
            a.mb = stage_in(c, S_V_MB, b->move_batch + i * b->move_stride, (size_t)D, host, &err);
            a.ev = c->dev<unsigned long long>(S_V_EV, (size_t)2 * D + 1);
            a.bcnt = c->dev<int32_t>(S_V_BCNT, (size_t)a.nb + 1);
            a.bmin = c->dev<int32_t>(S_V_BMIN, (size_t)a.nb + 1);
            a.bmax = c->dev<int32_t>(S_V_BMAX, (size_t)a.nb + 1);
            if (err != cudaSuccess || !a.ev || !a.bcnt || !a.bmin || !a.bmax)
                return cuda_fail(err != cudaSuccess ? err : cudaErrorMemoryAllocation, "validate batches", detail);
            CK(cudaMemsetAsync(a.bcnt, 0, ((size_t)a.nb + 1) * 4, c->stream), "memset");
            k_fill_i32<<<blocks_for(a.nb + 1, sms), 256, 0, c->stream>>>(a.bmin, a.nb + 1, INT_MAX);
            k_fill_i32<<<blocks_for(a.nb + 1, sms), 256, 0, c->stream>>>(a.bmax, a.nb + 1, INT_MIN);
        }
        // dag edges
        const int32_t *ea = nullptr, *eb = nullptr;
        int64_t ne = 0;
        if (b->dag_mode == RECON_DAG_EXPLICIT) {
            ne = eoff[i + 1] - eoff[i];
            ea = stage_in(c, S_EA, b->dag_a + eoff[i], (size_t)ne, host, &err);
            eb = stage_in(c, S_EB, b->dag_b + eoff[i], (size_t)ne, host, &err);
            if (err != cudaSuccess) return cuda_fail(err, "validate dag", detail);
        }
        if (b->dag_mode == RECON_DAG_OCCUPANCY) k_walk<true><<<blocks_for(P, sms), 256, 0, c->stream>>>(a);
        else k_walk<false><<<blocks_for(P, sms), 256, 0, c->stream>>>(a);
        if (ne) k_edges<<<blocks_for(ne, sms), 256, 0, c->stream>>>(a, ea, eb, ne);
        c->launches += 7;
        if (a.mb) {
            const int64_t ne2 = 2 * D;
            unsigned long long *sorted = c->dev<unsigned long long>(S_V_EV2, (size_t)ne2 + 1);
            size_t sb = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, sb, a.ev, sorted, (int)ne2, 0, 64, c->stream);
            void *stemp = c->get(S_TEMP, sb);
            if (!sorted || !stemp) return cuda_fail(cudaErrorMemoryAllocation, "validate sort", detail);
            CK(cub::DeviceRadixSort::SortKeys(stemp, sb, a.ev, sorted, (int)ne2, 0, 64, c->stream), "sort");
            k_events<<<blocks_for(ne2, sms), 256, 0, c->stream>>>(a, sorted, ne2);
            k_batches<<<blocks_for(a.nb, sms), 256, 0, c->stream>>>(a);
            c->launches += 3;
        }
        k_targets<<<blocks_for((int64_t)W * b->h_prime, sms), 256, 0, c->stream>>>(a);
        // rare paths: back edges (cycle check) and collisions / shared
        // endpoints (exact token replay)
        VState hs;
        CK(cudaMemcpyAsync(&hs, st, sizeof(VState), cudaMemcpyDeviceToHost, c->stream), "D2H");
        CK(cudaStreamSynchronize(c->stream), "D2H");
        if ((hs.raw & F_EDGE_BACK) && !(hs.raw & F_BOUNDS)) {
            if (b->dag_mode == RECON_DAG_OCCUPANCY) {  // materialise the implicit edges
                int64_t *cnt = c->dev<int64_t>(S_V_ECNT, (size_t)P + 1);
                if (!cnt) return cuda_fail(cudaErrorMemoryAllocation, "validate dag", detail);
                CK(cudaMemsetAsync(cnt + P, 0, 8, c->stream), "memset");
                k_occ_edges<false><<<blocks_for(P, sms), 256, 0, c->stream>>>(a, cnt, nullptr, nullptr);
                size_t t2 = 0;
                cub::DeviceScan::ExclusiveSum(nullptr, t2, cnt, cnt, P + 1, c->stream);
                void *tmp2 = c->get(S_TEMP, t2);
                if (!tmp2) return cuda_fail(cudaErrorMemoryAllocation, "validate dag", detail);
                CK(cub::DeviceScan::ExclusiveSum(tmp2, t2, cnt, cnt, P + 1, c->stream), "scan");
                CK(cudaMemcpyAsync(&ne, cnt + P, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
                CK(cudaStreamSynchronize(c->stream), "D2H");
                int32_t *xa = c->dev<int32_t>(S_EA, (size_t)ne + 1), *xb = c->dev<int32_t>(S_EB, (size_t)ne + 1);
                if (!xa || !xb) return cuda_fail(cudaErrorMemoryAllocation, "validate dag", detail);
                k_occ_edges<true><<<blocks_for(P, sms), 256, 0, c->stream>>>(a, cnt, xa, xb);
                ea = xa;
                eb = xb;
            }
            int8_t *alive = c->dev<int8_t>(S_V_ALIVE, (size_t)P + 1), *haspred = c->dev<int8_t>(S_V_PRED, (size_t)P + 1);
            if (!alive || !haspred) return cuda_fail(cudaErrorMemoryAllocation, "validate dag", detail);
            CK(cudaMemsetAsync(alive, 1, (size_t)P + 1, c->stream), "memset");
            CK(cudaMemsetAsync(haspred, 0, (size_t)P + 1, c->stream), "memset");
            for (;;) {
                hs.changed = hs.alive = 0;
                CK(cudaMemcpyAsync(&st->changed, &hs.changed, 8, cudaMemcpyHostToDevice, c->stream), "H2D");
                k_peel_mark<<<blocks_for(ne, sms), 256, 0, c->stream>>>(a, ea, eb, ne, alive, haspred);
                k_peel_remove<<<blocks_for(P, sms), 256, 0, c->stream>>>(a, alive, haspred);
                c->launches += 2;
                CK(cudaMemcpyAsync(&hs.changed, &st->changed, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
                CK(cudaStreamSynchronize(c->stream), "D2H");
                if (!hs.changed) break;
            }
            if (hs.alive) {
                hs.raw |= F_CYCLE;
                CK(cudaMemcpyAsync(&st->raw, &hs.raw, 4, cudaMemcpyHostToDevice, c->stream), "H2D");
            }
        }
        if ((hs.raw & (F_EXEC | F_SHARED_S | F_SHARED_T)) && !(hs.raw & F_BOUNDS)) {
            int32_t *buf = c->dev<int32_t>(S_V_TOK, (size_t)3 * V + 3 * (size_t)P + 1);
            int8_t *began = c->dev<int8_t>(S_V_BEGAN, (size_t)V);
            if (!buf || !began) return cuda_fail(cudaErrorMemoryAllocation, "validate tokens", detail);
            hs.tok_empty = hs.tok_second = INT_MAX;
            CK(cudaMemcpyAsync(&st->tok_empty, &hs.tok_empty, 8, cudaMemcpyHostToDevice, c->stream), "H2D");
            k_token_replay<<<1, 1, 0, c->stream>>>(a, buf, began);
            c->launches += 1;
        }
        k_verdict<<<1, 1, 0, c->stream>>>(st, ctd, cdp, b->move_batch != nullptr, a.nb, d_verdict + i);
        c->launches += 2;
        CK(cudaGetLastError(), "validate launch");
    }
    if (host) {
        CK(cudaMemcpyAsync(b->verdict, d_verdict, (size_t)n * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        CK(cudaStreamSynchronize(c->stream), "D2H");
    }
    return RECON_OK;
}

}  // namespace

extern "C" {

recon_status recon_validate_batch_run(recon_ctx *ctx, const recon_validate_batch *batch) {
    return validate_impl(ctx, batch, false);
}

recon_status recon_validate_batch_run_host(recon_ctx *ctx, const recon_validate_batch *batch) {
    return validate_impl(ctx, batch, true);
}

}  // extern "C"
