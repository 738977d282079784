/*
 * oracle/recon_oracle.c — TEST INFRASTRUCTURE (the CPU oracle), not product code.
 *
 * A plain-C restatement of the reference's hot path (arXiv 2504.06182
 * reference, /root/reference/proj) exposed behind the same C-ABI as the B200
 * library (include/recon_b200.h).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as a checker.
 *
 * It restates the algorithms in the form the GPU kernels use, so a parity
 * failure can be localised:
 *   - grid events are solved with the SPLIT RULE:
 *     residents always used, a = number of top-side tokens used, cost(a)
 *     convex, ties -> largest a.  This is the reference's window_dp tie rule
 *     (lex-min use vector read from the last source, exact1d.cpp:155-207)
 *     specialised to band targets;
 *   - red-rec / bird drivers follow redrec.cpp:124-232 and bird.cpp:54-123
 *     with column state held as depth bitmasks;
 *   - chains follow exact1d.cpp:219-407 (candidate / certified blocks) with a
 *     generic window DP restating exact1d.cpp:155-207 (ties -> smallest use);
 *   - batching follows batching.cpp:28-159 literally (ascending-id scan).
 *
 * Parity of this restatement is pinned against the compiled reference
 * (oracle/_ref/librecon_ref.so, built from the reference's own sources by
 * oracle/Makefile) and against the reference tests' pinned values
 * (tests/golden/, tests/test_oracle_vs_reference.py).
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <math.h>

#include "recon_b200.h"
#include "recon_sim_rng.h"
#include "digest_cpu.h"

struct recon_ctx {
    int device;
};

#define INF64 (INT64_MAX / 4)

static void *xcalloc(size_t n, size_t sz) {
    void *p = calloc(n ? n : 1, sz ? sz : 1);
    if (!p) abort();
    return p;
}

static int wpc_of(int h) { return (h + 63) / 64; }

/* ======================================================================== */
/* Grid state (column tokens as depth bitmasks)                              */
/* ======================================================================== */

typedef struct {
    int W, H, k, lo, hi, wpd; /* band depths [lo, hi] (virtual_line.cpp:47-50) */
    uint64_t *dep;            /* [W*wpd] current tokens of each column, bit = depth */
    int *sigma;               /* surplus (virtual_line.cpp:53-59) */
    char *solved;
    int *mark_dest;           /* red-rec: receiver this column's parked tokens are marked for */
    uint64_t *mark;           /* [W*wpd] red-rec marks, bit = depth in the marking column */
    /* output */
    int32_t *psrc, *pdst, *pev;
    int64_t np, cap, total;
    int nevents;
    int status, detail;
} gstate;

static int getbit(const uint64_t *m, int d) { return (int)((m[d >> 6] >> (d & 63)) & 1ULL); }
static void setbit(uint64_t *m, int d) { m[d >> 6] |= 1ULL << (d & 63); }
static void clrbit(uint64_t *m, int d) { m[d >> 6] &= ~(1ULL << (d & 63)); }

static int gstate_init(gstate *g, const uint64_t *occ, int W, int H, int hp) {
    memset(g, 0, sizeof(*g));
    g->W = W;
    g->H = H;
    g->k = hp;
    g->wpd = wpc_of(H);
    /* centered band rows y in [(H-h')/2, +h'-1] (problem.hpp:71-86) -> depths */
    int ylo = (H - hp) / 2, yhi = ylo + hp - 1;
    g->lo = H - 1 - yhi;
    g->hi = H - 1 - ylo;
    g->dep = xcalloc((size_t)W * g->wpd, 8);
    g->mark = xcalloc((size_t)W * g->wpd, 8);
    g->sigma = xcalloc((size_t)W, sizeof(int));
    g->solved = xcalloc((size_t)W, 1);
    g->mark_dest = xcalloc((size_t)W, sizeof(int));
    int wpc = wpc_of(H);
    long total = 0;
    for (int x = 0; x < W; ++x) {
        int cnt = 0;
        for (int y = 0; y < H; ++y)
            if ((occ[(size_t)x * wpc + y / 64] >> (y % 64)) & 1ULL) {
                setbit(g->dep + (size_t)x * g->wpd, H - 1 - y);
                ++cnt;
            }
        g->sigma[x] = cnt - hp;
        g->mark_dest[x] = -1;
        total += cnt;
    }
    if (hp <= 0 || hp >= H) return RECON_D_BAND_HEIGHT;
    if (total < (long)W * hp) return RECON_D_FEWER_SOURCES;
    return 0;
}

static void gstate_free(gstate *g) {
    free(g->dep);
    free(g->mark);
    free(g->sigma);
    free(g->solved);
    free(g->mark_dest);
}

/* One candidate token of an event (virtual_line.hpp:41-48). */
typedef struct {
    int64_t vpos;
    int dist, col, depth;
    int mand;
    int used;
} tok_t;

static int64_t vpos_of(const gstate *g, int depth, int dist) {
    /* virtual_line.cpp:65-68: dist 0 -> depth; top side depth-dist; else depth+dist */
    if (dist == 0) return depth;
    return depth < g->lo ? depth - dist : depth + dist;
}

static void add_token(const gstate *g, tok_t *t, int *n, int col, int depth, int recv, int mand) {
    int dist = col > recv ? col - recv : recv - col;
    tok_t *x = &t[(*n)++];
    x->vpos = vpos_of(g, depth, dist);
    x->dist = dist;
    x->col = col;
    x->depth = depth;
    x->mand = mand;
    x->used = 0;
}

/* group order: (pos, dist, column, vertex) — virtual_line.cpp:112-118 */
static int cmp_group(const void *pa, const void *pb) {
    const tok_t *a = pa, *b = pb;
    if (a->vpos != b->vpos) return a->vpos < b->vpos ? -1 : 1;
    if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
    if (a->col != b->col) return a->col < b->col ? -1 : 1;
    return a->depth - b->depth;
}

/* top-side preference: nearest to the band first (vpos desc), then group order */
static int cmp_top_pref(const void *pa, const void *pb) {
    const tok_t *a = *(const tok_t *const *)pa, *b = *(const tok_t *const *)pb;
    if (a->vpos != b->vpos) return a->vpos > b->vpos ? -1 : 1;
    if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
    return a->col - b->col;
}

static int cmp_bot_pref(const void *pa, const void *pb) {
    const tok_t *a = *(const tok_t *const *)pa, *b = *(const tok_t *const *)pb;
    if (a->vpos != b->vpos) return a->vpos < b->vpos ? -1 : 1;
    if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
    return a->col - b->col;
}

/*
 * Split-rule solve of one band event (equivalent to
 * assign_1d_generalized over build_virtual_event's instance,
 * exact1d.cpp:374-407 + virtual_line.cpp:97-142).  Marks tokens used.
 * Returns 0 or an INFEASIBLE detail code.
 */
static int split_solve(const gstate *g, tok_t *t, int n) {
    const int lo = g->lo, hi = g->hi, k = g->k;
    int R = 0, m_top = 0, m_bot = 0, n_ot = 0, n_ob = 0;
    int64_t sum_mtop = 0, sum_mbot = 0;
    tok_t **ot = xcalloc((size_t)n, sizeof(tok_t *));
    tok_t **ob = xcalloc((size_t)n, sizeof(tok_t *));
    int64_t *e = xcalloc((size_t)n, 8);
    int supply = 0, mandatory = 0;
    /* residents in depth order */
    qsort(t, (size_t)n, sizeof(tok_t), cmp_group);
    for (int i = 0; i < n; ++i) {
        ++supply;
        if (t[i].mand) ++mandatory;
        if (t[i].vpos >= lo && t[i].vpos <= hi) {
            /* residents are always mandatory (own band cells, virtual_line.cpp:92) */
            e[R] = t[i].vpos - lo - R;
            ++R;
        } else if (t[i].vpos < lo) {
            if (t[i].mand) {
                ++m_top;
                sum_mtop += t[i].vpos;
            } else {
                ot[n_ot++] = &t[i];
            }
        } else {
            if (t[i].mand) {
                ++m_bot;
                sum_mbot += t[i].vpos;
            } else {
                ob[n_ob++] = &t[i];
            }
        }
    }
    int rc = 0;
    if (supply < k) rc = RECON_D_GEN_SUPPLY;
    else if (mandatory > k) rc = RECON_D_GEN_MANDATORY;
    const int holes = k - R;
    int a_min = m_top, a_max = m_top + n_ot;
    if (holes - m_bot - n_ob > a_min) a_min = holes - m_bot - n_ob;
    if (holes - m_bot < a_max) a_max = holes - m_bot;
    if (!rc && a_min > a_max) rc = RECON_D_GEN_NO_ASSIGNMENT;
    if (rc) {
        free(ot);
        free(ob);
        free(e);
        return rc;
    }
    qsort(ot, (size_t)n_ot, sizeof(tok_t *), cmp_top_pref);
    qsort(ob, (size_t)n_ob, sizeof(tok_t *), cmp_bot_pref);
    int best_a = a_min;
    int64_t best = INF64;
    for (int a = a_min; a <= a_max; ++a) {
        const int b = holes - a;
        int64_t cost = (int64_t)a * lo + (int64_t)a * (a - 1) / 2 - sum_mtop;
        for (int j = 0; j < a - m_top; ++j) cost -= ot[j]->vpos;
        for (int r = 0; r < R; ++r) cost += e[r] > a ? e[r] - a : a - e[r];
        cost += sum_mbot - ((int64_t)b * hi - (int64_t)b * (b - 1) / 2);
        for (int j = 0; j < b - m_bot; ++j) cost += ob[j]->vpos;
        if (cost <= best) { /* ties -> largest a */
            best = cost;
            best_a = a;
        }
    }
    for (int i = 0; i < n; ++i) t[i].used = t[i].mand;
    for (int j = 0; j < best_a - m_top; ++j) ot[j]->used = 1;
    for (int j = 0; j < holes - best_a - m_bot; ++j) ob[j]->used = 1;
    free(ot);
    free(ob);
    free(e);
    return 0;
}

typedef struct {
    int64_t vpos, target;
    int col, depth;
} mover_t;

static int cmp_right(const void *pa, const void *pb) {
    const mover_t *a = pa, *b = pb;
    return a->target > b->target ? -1 : (a->target < b->target ? 1 : 0);
}
static int cmp_left(const void *pa, const void *pb) {
    const mover_t *a = pa, *b = pb;
    return a->target < b->target ? -1 : (a->target > b->target ? 1 : 0);
}

/*
 * Solve + realize one event (Runner::run / realize_event,
 * redrec.cpp:132-140, virtual_line.cpp:177-229): used tokens in group order
 * take band targets lo.. in order; movers emit in order_1d_intervals order
 * (rights by target desc, then lefts by target asc, exact1d.cpp:494-515).
 */
static int run_event(gstate *g, int recv, tok_t *t, int n) {
    int rc = split_solve(g, t, n);
    if (rc) return rc;
    /* t is sorted in group order by split_solve */
    mover_t *rights = xcalloc((size_t)g->k, sizeof(mover_t));
    mover_t *lefts = xcalloc((size_t)g->k, sizeof(mover_t));
    int nr = 0, nl = 0;
    int64_t target = g->lo;
    for (int i = 0; i < n; ++i) {
        if (!t[i].used) continue;
        mover_t m = {t[i].vpos, target, t[i].col, t[i].depth};
        if (target > t[i].vpos) rights[nr++] = m;
        else if (target < t[i].vpos) lefts[nl++] = m;
        ++target;
    }
    qsort(rights, (size_t)nr, sizeof(mover_t), cmp_right);
    qsort(lefts, (size_t)nl, sizeof(mover_t), cmp_left);
    for (int pass = 0; pass < 2; ++pass) {
        mover_t *arr = pass ? lefts : rights;
        int cnt = pass ? nl : nr;
        for (int i = 0; i < cnt; ++i) {
            if (g->np >= g->cap) {
                free(rights);
                free(lefts);
                return -1;
            }
            const int ys = g->H - 1 - arr[i].depth, yt = g->H - 1 - (int)arr[i].target;
            g->psrc[g->np] = arr[i].col * g->H + ys;
            g->pdst[g->np] = recv * g->H + yt;
            if (g->pev) g->pev[g->np] = g->nevents;
            int64_t len = arr[i].target - arr[i].vpos;
            g->total += len < 0 ? -len : len;
            ++g->np;
        }
    }
    free(rights);
    free(lefts);
    ++g->nevents;
    return 0;
}

static void set_band_only(gstate *g, int c) {
    uint64_t *m = g->dep + (size_t)c * g->wpd;
    memset(m, 0, (size_t)g->wpd * 8);
    for (int d = g->lo; d <= g->hi; ++d) setbit(m, d);
}

/* ---------------- red-rec (redrec.cpp) ---------------- */

static int own_tokens(const gstate *g, tok_t *t, int c) {
    int n = 0;
    const uint64_t *m = g->dep + (size_t)c * g->wpd;
    for (int d = 0; d < g->H; ++d)
        if (getbit(m, d)) add_token(g, t, &n, c, d, c, d >= g->lo && d <= g->hi);
    return n;
}

/* Runner::solve_own (redrec.cpp:144-165) */
static int rr_solve_own(gstate *g, tok_t *t, int c, int mark_receiver, int32_t *ev) {
    int n = own_tokens(g, t, c);
    if (ev) {
        int32_t *e = ev + 4 * g->nevents;
        e[0] = g->nevents;
        e[1] = c;
        e[2] = -1;
        e[3] = mark_receiver;
    }
    int rc = run_event(g, c, t, n);
    if (rc) return rc;
    uint64_t *m = g->dep + (size_t)c * g->wpd;
    set_band_only(g, c);
    if (mark_receiver >= 0) {
        uint64_t *mk = g->mark + (size_t)c * g->wpd;
        memset(mk, 0, (size_t)g->wpd * 8);
        for (int i = 0; i < n; ++i)
            if (!t[i].used) setbit(mk, t[i].depth);
        g->mark_dest[c] = mark_receiver;
        g->sigma[mark_receiver] += g->sigma[c];
        g->sigma[c] = 0;
    } else {
        for (int i = 0; i < n; ++i)
            if (!t[i].used) setbit(m, t[i].depth);
    }
    g->solved[c] = 1;
    return 0;
}

/* Runner::flush + build_redistribution_instance (redrec.cpp:92-116, 169-191) */
static int rr_flush(gstate *g, tok_t *t, int r, int d, int32_t *ev) {
    int n = 0;
    const uint64_t *mr = g->dep + (size_t)r * g->wpd;
    for (int dd = 0; dd < g->H; ++dd)
        if (getbit(mr, dd)) add_token(g, t, &n, r, dd, r, 1);
    for (int c = 0; c < g->W; ++c)
        if (g->mark_dest[c] == r) {
            const uint64_t *mk = g->mark + (size_t)c * g->wpd;
            for (int dd = 0; dd < g->H; ++dd)
                if (getbit(mk, dd)) add_token(g, t, &n, c, dd, r, 1);
        }
    const uint64_t *md = g->dep + (size_t)d * g->wpd;
    for (int dd = 0; dd < g->H; ++dd)
        if (getbit(md, dd) && (dd < g->lo || dd > g->hi)) add_token(g, t, &n, d, dd, r, 0);
    if (ev) {
        int32_t *e = ev + 4 * g->nevents;
        e[0] = g->nevents;
        e[1] = r;
        e[2] = d;
        e[3] = -1;
    }
    int rc = run_event(g, r, t, n);
    if (rc) return rc;
    int drawn = 0;
    for (int i = 0; i < n; ++i)
        if (t[i].used && !t[i].mand) {
            clrbit(g->dep + (size_t)d * g->wpd, t[i].depth);
            ++drawn;
        }
    g->sigma[d] -= drawn;
    for (int c = 0; c < g->W; ++c)
        if (g->mark_dest[c] == r) {
            g->mark_dest[c] = -1;
            memset(g->mark + (size_t)c * g->wpd, 0, (size_t)g->wpd * 8);
        }
    set_band_only(g, r);
    g->sigma[r] = 0;
    g->solved[r] = 1;
    return 0;
}

/* scan_for_donor (redrec.cpp:43-51) */
static int rr_scan(const gstate *g, int r, int step) {
    for (int c = r + step; c >= 0 && c < g->W; c += step) {
        if (!g->solved[c] && g->sigma[c] > 0) return c;
        if (g->solved[c] && g->sigma[c] == 0) continue;
        return -1;
    }
    return -1;
}

/* select_best_pair (redrec.cpp:55-86): key (-exchange, |d-r|, deficit-exchange, r, d) */
static int rr_select(const gstate *g, int *pd, int *pr) {
    int have_r = 0, have = 0;
    int bk[5] = {0, 0, 0, 0, 0};
    for (int r = 0; r < g->W; ++r) {
        if (g->solved[r] || g->sigma[r] >= 0) continue;
        have_r = 1;
        for (int side = 0; side < 2; ++side) {
            int d = rr_scan(g, r, side == 0 ? -1 : 1);
            if (d < 0) continue;
            int deficit = -g->sigma[r];
            int ex = g->sigma[d] < deficit ? g->sigma[d] : deficit;
            int key[5] = {-ex, d > r ? d - r : r - d, deficit - ex, r, d};
            int less = 0;
            if (have) {
                for (int q = 0; q < 5; ++q)
                    if (key[q] != bk[q]) {
                        less = key[q] < bk[q];
                        break;
                    }
            }
            if (!have || less) {
                memcpy(bk, key, sizeof(bk));
                have = 1;
            }
        }
    }
    if (!have_r) return RECON_D_NO_DEFICIT;
    if (!have) return RECON_D_NO_DONOR;
    *pd = bk[4];
    *pr = bk[3];
    return 0;
}

static int rr_deficit_remains(const gstate *g) {
    for (int c = 0; c < g->W; ++c)
        if (!g->solved[c] && g->sigma[c] < 0) return 1;
    return 0;
}

/* red_rec (redrec.cpp:205-232) */
static void redrec_run(gstate *g, int32_t *ev) {
    tok_t *t = xcalloc((size_t)g->W * g->H + 1, sizeof(tok_t));
    int rc = 0;
    for (int c = 0; c < g->W && !rc; ++c)
        if (g->sigma[c] == 0) rc = rr_solve_own(g, t, c, -1, ev);
    while (!rc && rr_deficit_remains(g)) {
        int d = -1, r = -1;
        int sel = rr_select(g, &d, &r);
        if (sel) {
            g->status = RECON_ERR_LOGIC;
            g->detail = sel;
            free(t);
            return;
        }
        const int ds = g->sigma[d], def = -g->sigma[r];
        if (ds < def) {
            rc = rr_solve_own(g, t, d, r, ev);
        } else {
            rc = rr_flush(g, t, r, d, ev);
            if (!rc && ds == def) rc = rr_solve_own(g, t, d, -1, ev);
        }
    }
    for (int c = 0; c < g->W && !rc; ++c)
        if (!g->solved[c]) rc = rr_solve_own(g, t, c, -1, ev);
    if (rc < 0) {
        g->status = RECON_ERR_CAPACITY;
    } else if (rc) {
        g->status = RECON_ERR_INFEASIBLE;
        g->detail = rc;
    }
    free(t);
}

/* ---------------- bird (bird.cpp) ---------------- */

/* BirdRunner::solve_column + build_generalized_instance (bird.cpp:35-46, 64-100) */
static int bird_column(gstate *g, tok_t *t, int c, int pooled, int32_t *order) {
    int n = own_tokens(g, t, c);
    if (pooled)
        for (int x = 0; x < g->W; ++x) {
            if (x == c) continue;
            const uint64_t *m = g->dep + (size_t)x * g->wpd;
            for (int d = 0; d < g->H; ++d)
                if (getbit(m, d) && (d < g->lo || d > g->hi)) add_token(g, t, &n, x, d, c, 0);
        }
    if (order) order[g->nevents] = c;
    int rc = run_event(g, c, t, n);
    if (rc) return rc;
    for (int i = 0; i < n; ++i)
        if (t[i].used && t[i].col != c) {
            clrbit(g->dep + (size_t)t[i].col * g->wpd, t[i].depth);
            --g->sigma[t[i].col];
        }
    set_band_only(g, c);
    int left = 0;
    for (int i = 0; i < n; ++i)
        if (!t[i].used && t[i].col == c) {
            setbit(g->dep + (size_t)c * g->wpd, t[i].depth);
            ++left;
        }
    g->sigma[c] = left;
    g->solved[c] = 1;
    return 0;
}

static void bird_run(gstate *g, int32_t *order) {
    tok_t *t = xcalloc((size_t)g->W * g->H + 1, sizeof(tok_t));
    int rc = 0;
    for (int c = 0; c < g->W && !rc; ++c)
        if (g->sigma[c] >= 0) rc = bird_column(g, t, c, 0, order);
    for (int c = 0; c < g->W && !rc; ++c)
        if (!g->solved[c]) rc = bird_column(g, t, c, 1, order);
    if (rc < 0) {
        g->status = RECON_ERR_CAPACITY;
    } else if (rc) {
        g->status = RECON_ERR_INFEASIBLE;
        g->detail = rc;
    }
    free(t);
}

/* ======================================================================== */
/* occupancy_dag (virtual_line.cpp:241-268)                                  */
/* ======================================================================== */

typedef struct {
    int32_t a, b;
} edge_t;

static int cmp_edge(const void *pa, const void *pb) {
    const edge_t *x = pa, *y = pb;
    if (x->a != y->a) return x->a < y->a ? -1 : 1;
    return x->b < y->b ? -1 : (x->b > y->b);
}

/* one-bend path walk: horizontal along the source row, then vertical (virtual_line.cpp:150-173) */
static int64_t walk_path(int H, int32_t s, int32_t t, int32_t *out) {
    int xs = s / H, ys = s % H, xt = t / H, yt = t % H;
    int64_t n = 0;
    int x = xs, y = ys;
    out[n++] = x * H + y;
    while (x != xt) {
        x += xt > x ? 1 : -1;
        out[n++] = x * H + y;
    }
    while (y != yt) {
        y += yt > y ? 1 : -1;
        out[n++] = x * H + y;
    }
    return n;
}

static int64_t dag_edges(int W, int H, const int32_t *ps, const int32_t *pt, int64_t np, edge_t **out) {
    int32_t *src_of = xcalloc((size_t)W * H, 4), *tgt_of = xcalloc((size_t)W * H, 4);
    for (int64_t v = 0; v < (int64_t)W * H; ++v) src_of[v] = tgt_of[v] = -1;
    for (int64_t i = 0; i < np; ++i) {
        src_of[ps[i]] = (int32_t)i;
        tgt_of[pt[i]] = (int32_t)i;
    }
    int64_t cap = 64, ne = 0;
    edge_t *e = xcalloc((size_t)cap, sizeof(edge_t));
    int32_t *verts = xcalloc((size_t)(W + H + 2), 4);
    for (int64_t i = 0; i < np; ++i) {
        int64_t nv = walk_path(H, ps[i], pt[i], verts);
        for (int64_t k = 0; k < nv; ++k) {
            int32_t v = verts[k];
            if (ne + 2 > cap) {
                cap *= 2;
                e = realloc(e, (size_t)cap * sizeof(edge_t));
            }
            if (src_of[v] >= 0 && src_of[v] != i) e[ne++] = (edge_t){src_of[v], (int32_t)i};
            if (tgt_of[v] >= 0 && tgt_of[v] != i) e[ne++] = (edge_t){(int32_t)i, tgt_of[v]};
        }
    }
    qsort(e, (size_t)ne, sizeof(edge_t), cmp_edge);
    int64_t u = 0;
    for (int64_t i = 0; i < ne; ++i)
        if (u == 0 || e[i].a != e[u - 1].a || e[i].b != e[u - 1].b) e[u++] = e[i];
    free(src_of);
    free(tgt_of);
    free(verts);
    *out = e;
    return u;
}

/* ======================================================================== */
/* C-ABI: grid                                                               */
/* ======================================================================== */

const char *recon_detail_message(int32_t detail) {
    (void)detail;
    return "";
}
const char *recon_last_cuda_error(void) { return ""; }
int32_t recon_abi_version(void) { return RECON_ABI_VERSION; }
recon_status recon_ctx_create(int32_t device, recon_ctx **out) {
    *out = xcalloc(1, sizeof(recon_ctx));
    (*out)->device = device;
    return RECON_OK;
}
void recon_ctx_destroy(recon_ctx *ctx) { free(ctx); }
void *recon_ctx_stream(recon_ctx *ctx) {
    (void)ctx;
    return NULL;
}
int64_t recon_ctx_launch_count(recon_ctx *ctx) {
    (void)ctx;
    return 0;
}
recon_status recon_ctx_set_kernel_timing(recon_ctx *ctx, int32_t enable) {
    (void)ctx;
    (void)enable;
    return RECON_OK;
}
recon_status recon_ctx_kernel_times(recon_ctx *ctx, float *ms, int32_t n) {
    (void)ctx;
    for (int32_t i = 0; i < n; ++i) ms[i] = 0.0f;
    return RECON_OK;
}

static recon_status grid_solve(int pooled, const uint64_t *occ, int W, int H, int hp,
                               recon_grid_solution *out, int32_t *detail) {
    if (detail) *detail = 0;
    if (W <= 0 || H <= 0) {
        if (detail) *detail = RECON_D_GRID_DIMENSIONS;
        return RECON_ERR_INPUT;
    }
    gstate g;
    int d0 = gstate_init(&g, occ, W, H, hp);
    if (d0) {
        gstate_free(&g);
        if (detail) *detail = d0;
        return d0 == RECON_D_FEWER_SOURCES ? RECON_ERR_INFEASIBLE : RECON_ERR_INPUT;
    }
    g.psrc = out->path_src;
    g.pdst = out->path_dst;
    g.pev = out->path_event;
    g.cap = out->path_capacity;
    int32_t *ev = xcalloc((size_t)W * 4, 4);
    if (pooled) bird_run(&g, ev);
    else redrec_run(&g, ev);
    recon_status st = (recon_status)g.status;
    if (detail) *detail = g.detail;
    out->path_count = g.np;
    out->displaced_tokens = g.np;
    out->total_displacement = g.total;
    out->event_count = g.nevents;
    if (st == RECON_OK && out->events) {
        int need = pooled ? g.nevents : 4 * g.nevents;
        if (need > out->event_capacity) st = RECON_ERR_CAPACITY;
        else memcpy(out->events, ev, (size_t)need * 4);
    }
    if (st == RECON_OK && out->dag_src) {
        edge_t *e = NULL;
        int64_t ne = dag_edges(W, H, out->path_src, out->path_dst, g.np, &e);
        out->dag_count = ne;
        if (ne > out->dag_capacity) {
            st = RECON_ERR_CAPACITY;
        } else {
            for (int64_t i = 0; i < ne; ++i) {
                out->dag_src[i] = e[i].a;
                out->dag_dst[i] = e[i].b;
            }
        }
        free(e);
    }
    free(ev);
    gstate_free(&g);
    return st;
}

recon_status recon_redrec_solve(recon_ctx *ctx, const uint64_t *occ, int32_t width, int32_t height,
                                int32_t h_prime, recon_grid_solution *out, int32_t *detail) {
    (void)ctx;
    return grid_solve(0, occ, width, height, h_prime, out, detail);
}

recon_status recon_bird_solve(recon_ctx *ctx, const uint64_t *occ, int32_t width, int32_t height,
                              int32_t h_prime, recon_grid_solution *out, int32_t *detail) {
    (void)ctx;
    return grid_solve(1, occ, width, height, h_prime, out, detail);
}

recon_status recon_occupancy_dag(recon_ctx *ctx, int32_t width, int32_t height,
                                 const int32_t *path_src, const int32_t *path_dst,
                                 int64_t path_count, int32_t *dag_src, int32_t *dag_dst,
                                 int64_t dag_capacity, int64_t *dag_count, int32_t *detail) {
    (void)ctx;
    if (detail) *detail = 0;
    edge_t *e = NULL;
    int64_t ne = dag_edges(width, height, path_src, path_dst, path_count, &e);
    *dag_count = ne;
    recon_status st = RECON_OK;
    if (ne > dag_capacity) st = RECON_ERR_CAPACITY;
    else
        for (int64_t i = 0; i < ne; ++i) {
            dag_src[i] = e[i].a;
            dag_dst[i] = e[i].b;
        }
    free(e);
    return st;
}

static recon_status grid_batch(int pooled, const recon_grid_batch *b) {
    const int wpc = wpc_of(b->height);
    const int64_t stride = (int64_t)b->width * b->h_prime;
    for (int i = 0; i < b->count; ++i) {
        recon_grid_solution out;
        memset(&out, 0, sizeof(out));
        out.path_src = b->path_src + i * stride;
        out.path_dst = b->path_dst + i * stride;
        out.path_event = b->path_event ? b->path_event + i * stride : NULL;
        out.path_capacity = stride;
        out.events = b->events ? b->events + (size_t)i * b->width * (pooled ? 1 : 4) : NULL;
        out.event_capacity = b->width * (pooled ? 1 : 4);
        int32_t det = 0;
        recon_status st = grid_solve(pooled, b->occ + (size_t)i * b->width * wpc, b->width, b->height,
                                     b->h_prime, &out, &det);
        b->status[i] = st;
        if (b->detail) b->detail[i] = det;
        b->path_count[i] = st == RECON_OK ? (int32_t)out.path_count : 0;
        b->total_displacement[i] = st == RECON_OK ? out.total_displacement : 0;
    }
    return RECON_OK;
}

recon_status recon_redrec_solve_batch(recon_ctx *c, const recon_grid_batch *b) {
    (void)c;
    return grid_batch(0, b);
}
recon_status recon_bird_solve_batch(recon_ctx *c, const recon_grid_batch *b) {
    (void)c;
    return grid_batch(1, b);
}
recon_status recon_redrec_solve_batch_host(recon_ctx *c, const recon_grid_batch *b) {
    (void)c;
    return grid_batch(0, b);
}
recon_status recon_bird_solve_batch_host(recon_ctx *c, const recon_grid_batch *b) {
    (void)c;
    return grid_batch(1, b);
}

/* *_batch_host_packed (include/recon_b200.h): the same solve, paths packed as
 * src | dst << 16 (grids of at most 65,536 cells). */
static recon_status grid_batch_packed(int pooled, const recon_grid_batch *b, uint32_t *packed) {
    if (!packed || !b) return RECON_ERR_ARGUMENT;
    if ((int64_t)b->width * b->height > 65536) return RECON_ERR_ARGUMENT;
    const size_t n = (size_t)(b->count > 0 ? b->count : 0) * (size_t)b->width * (size_t)b->h_prime;
    recon_grid_batch t = *b;
    t.path_src = (int32_t *)malloc((n ? n : 1) * sizeof(int32_t));
    t.path_dst = (int32_t *)malloc((n ? n : 1) * sizeof(int32_t));
    recon_status st = RECON_ERR_ARGUMENT;
    if (t.path_src && t.path_dst) {
        memset(t.path_src, 0, (n ? n : 1) * sizeof(int32_t));
        memset(t.path_dst, 0, (n ? n : 1) * sizeof(int32_t));
        st = grid_batch(pooled, &t);
        for (size_t i = 0; i < n; ++i) packed[i] = (uint32_t)t.path_src[i] | (uint32_t)t.path_dst[i] << 16;
    }
    free(t.path_src);
    free(t.path_dst);
    return st;
}
recon_status recon_redrec_solve_batch_host_packed(recon_ctx *c, const recon_grid_batch *b, uint32_t *packed) {
    (void)c;
    return grid_batch_packed(0, b, packed);
}
recon_status recon_bird_solve_batch_host_packed(recon_ctx *c, const recon_grid_batch *b, uint32_t *packed) {
    (void)c;
    return grid_batch_packed(1, b, packed);
}

/* ======================================================================== */
/* Exact 1D (exact1d.cpp)                                                    */
/* ======================================================================== */

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return x < y ? -1 : (x > y);
}

/*
 * Window DP (exact1d.cpp:155-207): sources (pos, lo, hi) ascending, targets
 * ascending; each source serves a consecutive run of u targets, lo <= u <= hi.
 * Among optimal use vectors returns the lexicographically smallest read from
 * the last source (per row: smallest feasible run among ties).  Returns 0 and
 * fills use[] / *weight, or -1 when infeasible.
 */
static int window_dp(int p, const int64_t *pos, const int32_t *lo, const int32_t *hi, int k,
                     const int64_t *tgt, int32_t *use, int64_t *weight) {
    int64_t *prev = xcalloc((size_t)k + 1, 8), *cur = xcalloc((size_t)k + 1, 8);
    int64_t *c = xcalloc((size_t)k + 1, 8);
    int32_t *choice = xcalloc((size_t)p * (k + 1) + 1, 4);
    for (int j = 0; j <= k; ++j) prev[j] = INF64;
    prev[0] = 0;
    for (int i = 0; i < p; ++i) {
        c[0] = 0;
        for (int j = 1; j <= k; ++j) {
            int64_t d = pos[i] - tgt[j - 1];
            c[j] = c[j - 1] + (d < 0 ? -d : d);
        }
        for (int j = 0; j <= k; ++j) {
            int64_t best = INF64;
            int bs = 0;
            for (int s = lo[i]; s <= hi[i] && s <= j; ++s) {
                if (prev[j - s] >= INF64) continue;
                int64_t v = prev[j - s] + c[j] - c[j - s];
                if (v < best) {
                    best = v;
                    bs = s;
                }
            }
            cur[j] = best;
            choice[(size_t)i * (k + 1) + j] = bs;
        }
        int64_t *tmp = prev;
        prev = cur;
        cur = tmp;
    }
    int rc = 0;
    if (prev[k] >= INF64) {
        rc = -1;
    } else {
        *weight = prev[k];
        int j = k;
        for (int i = p - 1; i >= 0; --i) {
            int s = choice[(size_t)i * (k + 1) + j];
            use[i] = s;
            j -= s;
        }
    }
    free(prev);
    free(cur);
    free(c);
    free(choice);
    return rc;
}

/* exact optimum of 0/1 sources onto targets (stands in for certifier_cost, exact1d.cpp:106-136) */
static int64_t line_cost(int ns, const int32_t *S, int nt, const int32_t *T) {
    if (nt == 0) return 0;
    int64_t *pos = xcalloc((size_t)ns, 8), *tg = xcalloc((size_t)nt, 8);
    int32_t *lo = xcalloc((size_t)ns, 4), *hi = xcalloc((size_t)ns, 4), *use = xcalloc((size_t)ns, 4);
    for (int i = 0; i < ns; ++i) {
        pos[i] = S[i];
        hi[i] = 1;
    }
    for (int i = 0; i < nt; ++i) tg[i] = T[i];
    int64_t w = INF64;
    window_dp(ns, pos, lo, hi, nt, tg, use, &w);
    free(pos);
    free(tg);
    free(lo);
    free(hi);
    free(use);
    return w;
}

typedef struct {
    int s0, s1, t0, t1; /* [s0,s1) slice of sorted S, [t0,t1) slice of sorted T */
} block_t;

/* candidate_blocks (exact1d.cpp:219-247) */
static int candidate_blocks(int n, int ns, const int32_t *S, int nt, const int32_t *T, block_t *out) {
    char *is_s = xcalloc((size_t)n, 1), *is_t = xcalloc((size_t)n, 1);
    int *suf_s = xcalloc((size_t)n + 1, sizeof(int)), *suf_t = xcalloc((size_t)n + 1, sizeof(int));
    for (int i = 0; i < ns; ++i) is_s[S[i]] = 1;
    for (int i = 0; i < nt; ++i) is_t[T[i]] = 1;
    for (int v = n - 1; v >= 0; --v) {
        suf_s[v] = suf_s[v + 1] + is_s[v];
        suf_t[v] = suf_t[v + 1] + is_t[v];
    }
    int nb = 0, si = 0, ti = 0;
    block_t cur = {0, 0, 0, 0};
    for (int v = 0; v < n; ++v) {
        if (is_s[v] || is_t[v]) {
            if (is_s[v]) cur.s1 = ++si;
            if (is_t[v]) cur.t1 = ++ti;
            continue;
        }
        if (cur.s1 - cur.s0 >= cur.t1 - cur.t0 && suf_s[v] >= suf_t[v]) {
            if (cur.s1 > cur.s0 || cur.t1 > cur.t0) out[nb++] = cur;
            cur.s0 = cur.s1 = si;
            cur.t0 = cur.t1 = ti;
        }
    }
    if (cur.s1 > cur.s0 || cur.t1 > cur.t0) out[nb++] = cur;
    free(is_s);
    free(is_t);
    free(suf_s);
    free(suf_t);
    return nb;
}

/* certified_blocks (exact1d.cpp:255-297) */
static int certified_blocks(int n, int ns, const int32_t *S, int nt, const int32_t *T, block_t *b) {
    int nb = candidate_blocks(n, ns, S, nt, T, b);
    if (nb <= 1) return nb;
    int64_t global = line_cost(ns, S, nt, T);
    int64_t *w = xcalloc((size_t)nb, 8);
    int64_t sum = 0;
    for (int i = 0; i < nb; ++i) {
        w[i] = line_cost(b[i].s1 - b[i].s0, S + b[i].s0, b[i].t1 - b[i].t0, T + b[i].t0);
        sum += w[i];
    }
    if (sum == global) {
        free(w);
        return nb;
    }
    int i = 0;
    while (i + 1 < nb) {
        block_t j = {b[i].s0, b[i + 1].s1, b[i].t0, b[i + 1].t1};
        int64_t wj = line_cost(j.s1 - j.s0, S + j.s0, j.t1 - j.t0, T + j.t0);
        if (wj < w[i] + w[i + 1]) {
            b[i] = j;
            w[i] = wj;
            memmove(b + i + 1, b + i + 2, (size_t)(nb - i - 2) * sizeof(block_t));
            memmove(w + i + 1, w + i + 2, (size_t)(nb - i - 2) * 8);
            --nb;
            if (i > 0) --i;
        } else {
            ++i;
        }
    }
    sum = 0;
    for (int q = 0; q < nb; ++q) sum += w[q];
    free(w);
    if (sum == global) return nb;
    b[0] = (block_t){0, ns, 0, nt};
    return 1;
}

/* validate_chain_instance (exact1d.cpp:299-312) on sorted inputs */
static recon_status validate_chain(int n, int ns, const int32_t *S, int nt, const int32_t *T, int32_t *detail) {
    if (n <= 0) {
        *detail = RECON_D_CHAIN_LENGTH;
        return RECON_ERR_INPUT;
    }
    for (int pass = 0; pass < 2; ++pass) {
        const int32_t *v = pass ? T : S;
        int cnt = pass ? nt : ns;
        for (int i = 0; i < cnt; ++i) {
            if (v[i] < 0 || v[i] >= n) {
                *detail = pass ? RECON_D_TARGET_OOB : RECON_D_SOURCE_OOB;
                return RECON_ERR_INPUT;
            }
            if (i > 0 && v[i] <= v[i - 1]) {
                *detail = pass ? RECON_D_TARGET_ORDER : RECON_D_SOURCE_ORDER;
                return RECON_ERR_INPUT;
            }
        }
    }
    if (ns < nt) {
        *detail = RECON_D_FEWER_SOURCES;
        return RECON_ERR_INFEASIBLE;
    }
    return RECON_OK;
}

/* assign_1d (exact1d.cpp:342-372) on sorted copies; pairs sorted by target */
static recon_status assign_1d_sorted(int n, int ns, int32_t *S, int nt, int32_t *T, int64_t *weight,
                                     int64_t *ps, int64_t *pt, int32_t *use, int32_t *detail) {
    qsort(S, (size_t)ns, 4, cmp_i32);
    qsort(T, (size_t)nt, 4, cmp_i32);
    recon_status st = validate_chain(n, ns, S, nt, T, detail);
    if (st) return st;
    *weight = 0;
    for (int i = 0; i < ns; ++i) use[i] = 0;
    if (nt == 0) return RECON_OK;
    block_t *b = xcalloc((size_t)ns + nt + 2, sizeof(block_t));
    int nb = certified_blocks(n, ns, S, nt, T, b);
    int np = 0;
    for (int q = 0; q < nb; ++q) {
        int bs = b[q].s1 - b[q].s0, bt = b[q].t1 - b[q].t0;
        if (bt == 0) continue;
        int64_t *pos = xcalloc((size_t)bs, 8), *tg = xcalloc((size_t)bt, 8);
        int32_t *lo = xcalloc((size_t)bs, 4), *hi = xcalloc((size_t)bs, 4);
        for (int i = 0; i < bs; ++i) {
            pos[i] = S[b[q].s0 + i];
            hi[i] = 1;
        }
        for (int i = 0; i < bt; ++i) tg[i] = T[b[q].t0 + i];
        int64_t w = 0;
        window_dp(bs, pos, lo, hi, bt, tg, use + b[q].s0, &w);
        *weight += w;
        int tp = 0;
        for (int i = 0; i < bs; ++i)
            if (use[b[q].s0 + i] > 0) {
                ps[np] = S[b[q].s0 + i];
                pt[np] = tg[tp++];
                ++np;
            }
        free(pos);
        free(tg);
        free(lo);
        free(hi);
    }
    free(b);
    return RECON_OK;
}

recon_status recon_assign_1d(recon_ctx *ctx, int32_t n, const int32_t *S, int32_t ns, const int32_t *T,
                             int32_t nt, int64_t *weight, int64_t *pair_src, int64_t *pair_dst,
                             int32_t *use_count, int32_t *detail) {
    (void)ctx;
    int32_t det = 0;
    int32_t *s = xcalloc((size_t)ns, 4), *t = xcalloc((size_t)nt, 4);
    memcpy(s, S, (size_t)ns * 4);
    memcpy(t, T, (size_t)nt * 4);
    recon_status st = assign_1d_sorted(n, ns, s, nt, t, weight, pair_src, pair_dst, use_count, &det);
    if (detail) *detail = det;
    free(s);
    free(t);
    return st;
}

recon_status recon_assign_1d_generalized(recon_ctx *ctx, int32_t nsrc, const int64_t *pos,
                                         const int32_t *multiplicity, const int32_t *min_use,
                                         int32_t nt, const int64_t *targets, int64_t *weight,
                                         int64_t *pair_src, int64_t *pair_dst, int32_t *use_count,
                                         int32_t *detail) {
    (void)ctx;
    int32_t det = 0;
    int64_t supply = 0, mand = 0;
    recon_status st = RECON_OK;
    /* checks in the reference's order (exact1d.cpp:374-396) */
    for (int i = 0; i < nsrc && !st; ++i) {
        if (multiplicity[i] < 1) {
            det = RECON_D_GEN_MULTIPLICITY;
            st = RECON_ERR_INPUT;
        } else if (min_use[i] < 0 || min_use[i] > multiplicity[i]) {
            det = RECON_D_GEN_MIN_USE;
            st = RECON_ERR_INPUT;
        } else if (i > 0 && pos[i] <= pos[i - 1]) {
            det = RECON_D_GEN_SOURCE_ORDER;
            st = RECON_ERR_INPUT;
        }
        supply += multiplicity[i];
        mand += min_use[i];
    }
    for (int i = 1; i < nt && !st; ++i)
        if (targets[i] <= targets[i - 1]) {
            det = RECON_D_GEN_TARGET_ORDER;
            st = RECON_ERR_INPUT;
        }
    if (!st && supply < nt) {
        det = RECON_D_GEN_SUPPLY;
        st = RECON_ERR_INFEASIBLE;
    }
    if (!st && mand > nt) {
        det = RECON_D_GEN_MANDATORY;
        st = RECON_ERR_INFEASIBLE;
    }
    if (!st) {
        if (window_dp(nsrc, pos, min_use, multiplicity, nt, targets, use_count, weight)) {
            det = RECON_D_GEN_NO_ASSIGNMENT;
            st = RECON_ERR_INFEASIBLE;
        } else {
            int tp = 0;
            for (int i = 0; i < nsrc; ++i)
                for (int u = 0; u < use_count[i]; ++u) {
                    pair_src[tp] = pos[i];
                    pair_dst[tp] = targets[tp];
                    ++tp;
                }
        }
    }
    if (detail) *detail = det;
    return st;
}

typedef struct {
    int64_t lo, hi;
    int id, rank;
    int64_t seq;
} span_t;

static int cmp_span_sweep(const void *pa, const void *pb) {
    const span_t *a = pa, *b = pb;
    if (a->lo != b->lo) return a->lo < b->lo ? -1 : 1;
    return a->id - b->id;
}

/* order_1d_intervals (exact1d.cpp:494-515) */
static void order_intervals(int np, const int32_t *s, const int32_t *t, int32_t *order) {
    int k = 0;
    /* rights by target desc (targets distinct), lefts by target asc, isolated by index */
    int32_t *r = xcalloc((size_t)np, 4), *l = xcalloc((size_t)np, 4);
    int nr = 0, nl = 0;
    for (int i = 0; i < np; ++i) {
        if (t[i] > s[i]) r[nr++] = i;
        else if (t[i] < s[i]) l[nl++] = i;
    }
    for (int i = 1; i < nr; ++i)
        for (int j = i; j > 0 && t[r[j]] > t[r[j - 1]]; --j) {
            int32_t x = r[j];
            r[j] = r[j - 1];
            r[j - 1] = x;
        }
    for (int i = 1; i < nl; ++i)
        for (int j = i; j > 0 && t[l[j]] < t[l[j - 1]]; --j) {
            int32_t x = l[j];
            l[j] = l[j - 1];
            l[j - 1] = x;
        }
    for (int i = 0; i < nr; ++i) order[k++] = r[i];
    for (int i = 0; i < nl; ++i) order[k++] = l[i];
    for (int i = 0; i < np; ++i)
        if (t[i] == s[i]) order[k++] = i;
    free(r);
    free(l);
}

recon_status recon_solve_1d(recon_ctx *ctx, int32_t n, const int32_t *S, int32_t ns, const int32_t *T,
                            int32_t nt, int32_t *path_src, int32_t *path_dst, int32_t *path_order,
                            int32_t *dag_src, int32_t *dag_dst, int64_t dag_capacity,
                            int64_t *dag_count, int64_t *total_displacement, int32_t *displaced,
                            int32_t *detail) {
    (void)ctx;
    int64_t w = 0;
    int64_t *ps = xcalloc((size_t)nt + 1, 8), *pt = xcalloc((size_t)nt + 1, 8);
    int32_t *use = xcalloc((size_t)ns + 1, 4);
    recon_status st = recon_assign_1d(NULL, n, S, ns, T, nt, &w, ps, pt, use, detail);
    if (st) {
        free(ps);
        free(pt);
        free(use);
        return st;
    }
    /* paths_from_matching + resolve_nesting (exact1d.cpp:430-492): re-pair each
       orientation class by sorted order */
    int32_t *s = xcalloc((size_t)nt + 1, 4), *t = xcalloc((size_t)nt + 1, 4);
    for (int i = 0; i < nt; ++i) {
        s[i] = (int32_t)ps[i];
        t[i] = (int32_t)pt[i];
    }
    for (int cls = 0; cls < 2; ++cls) {
        int32_t *ids = xcalloc((size_t)nt + 1, 4), *ss = xcalloc((size_t)nt + 1, 4), *tt = xcalloc((size_t)nt + 1, 4);
        int m = 0;
        for (int i = 0; i < nt; ++i)
            if (cls == 0 ? t[i] > s[i] : t[i] < s[i]) {
                ids[m] = i;
                ss[m] = s[i];
                tt[m] = t[i];
                ++m;
            }
        qsort(ss, (size_t)m, 4, cmp_i32);
        qsort(tt, (size_t)m, 4, cmp_i32);
        /* ids ordered by source (asc for rights, desc for lefts), paired with
           sorted sources/targets in the same direction */
        for (int i = 1; i < m; ++i)
            for (int j = i; j > 0 && s[ids[j]] < s[ids[j - 1]]; --j) {
                int32_t x = ids[j];
                ids[j] = ids[j - 1];
                ids[j - 1] = x;
            }
        for (int q = 0; q < m; ++q) {
            s[ids[q]] = ss[q];
            t[ids[q]] = tt[q];
        }
        free(ids);
        free(ss);
        free(tt);
    }
    int64_t total = 0;
    int disp = 0;
    for (int i = 0; i < nt; ++i) {
        path_src[i] = s[i];
        path_dst[i] = t[i];
        total += s[i] > t[i] ? s[i] - t[i] : t[i] - s[i];
        disp += s[i] != t[i];
    }
    *total_displacement = total;
    *displaced = disp;
    int32_t *order = xcalloc((size_t)nt + 1, 4);
    order_intervals(nt, s, t, order);
    if (path_order) memcpy(path_order, order, (size_t)nt * 4);
    /* span-overlap DAG in the reference's emission order (exact1d.cpp:529-560):
       sweep by (lo, id); active spans iterated by (hi, insertion order) */
    int32_t *rank = xcalloc((size_t)nt + 1, 4);
    for (int k = 0; k < nt; ++k) rank[order[k]] = k;
    span_t *sp = xcalloc((size_t)nt + 1, sizeof(span_t));
    for (int i = 0; i < nt; ++i) {
        sp[i].lo = s[i] < t[i] ? s[i] : t[i];
        sp[i].hi = s[i] < t[i] ? t[i] : s[i];
        sp[i].id = i;
    }
    qsort(sp, (size_t)nt, sizeof(span_t), cmp_span_sweep);
    span_t *act = xcalloc((size_t)nt + 1, sizeof(span_t));
    int na = 0;
    int64_t ne = 0;
    for (int q = 0; q < nt; ++q) {
        int drop = 0;
        while (drop < na && act[drop].hi < sp[q].lo) ++drop;
        memmove(act, act + drop, (size_t)(na - drop) * sizeof(span_t));
        na -= drop;
        for (int a = 0; a < na; ++a) {
            int other = act[a].id, me = sp[q].id;
            int x = rank[other] < rank[me] ? other : me;
            int y = x == other ? me : other;
            if (dag_src && ne < dag_capacity) {
                dag_src[ne] = x;
                dag_dst[ne] = y;
            }
            ++ne;
        }
        /* insert keeping (hi asc, insertion order) */
        int pos = na;
        while (pos > 0 && act[pos - 1].hi > sp[q].hi) --pos;
        memmove(act + pos + 1, act + pos, (size_t)(na - pos) * sizeof(span_t));
        act[pos] = sp[q];
        ++na;
    }
    if (dag_count) *dag_count = ne;
    if (dag_src && ne > dag_capacity) st = RECON_ERR_CAPACITY;
    free(rank);
    free(sp);
    free(act);
    free(order);
    free(s);
    free(t);
    free(ps);
    free(pt);
    free(use);
    return st;
}

static recon_status chain_batch(const recon_chain_batch *b) {
    const int wpn = (b->n + 63) / 64;
    const int nt = b->t_hi - b->t_lo + 1;
    int32_t *S = xcalloc((size_t)b->n + 1, 4), *T = xcalloc((size_t)nt + 1, 4);
    for (int i = 0; i < nt; ++i) T[i] = b->t_lo + i;
    for (int i = 0; i < b->count; ++i) {
        int ns = 0;
        const uint64_t *w = b->occ + (size_t)i * wpn;
        for (int v = 0; v < b->n; ++v)
            if ((w[v / 64] >> (v % 64)) & 1ULL) S[ns++] = v;
        int32_t det = 0, disp = 0;
        int64_t tot = 0;
        recon_status st = recon_solve_1d(NULL, b->n, S, ns, T, nt, b->path_src + (size_t)i * nt,
                                         b->path_dst + (size_t)i * nt, NULL, NULL, NULL, 0, NULL, &tot,
                                         &disp, &det);
        b->status[i] = st;
        if (b->detail) b->detail[i] = det;
        b->total_displacement[i] = tot;
        b->displaced[i] = disp;
    }
    free(S);
    free(T);
    return RECON_OK;
}

recon_status recon_solve_1d_batch(recon_ctx *c, const recon_chain_batch *b) {
    (void)c;
    return chain_batch(b);
}
recon_status recon_solve_1d_batch_host(recon_ctx *c, const recon_chain_batch *b) {
    (void)c;
    return chain_batch(b);
}

/* ======================================================================== */
/* Batching (batching.cpp:28-159)                                            */
/* ======================================================================== */

/* move_dir (batching.cpp:9-15): 0 up, 1 down, 2 left, 3 right */
static int move_dir(int H, int32_t a, int32_t b) {
    int ax = a / H, ay = a % H, bx = b / H, by = b % H;
    if (by > ay) return 0;
    if (by < ay) return 1;
    if (bx < ax) return 2;
    return 3;
}

static int compatible(int preset, int H, int32_t af, int32_t at, int32_t bf, int32_t bt) {
    if (preset == RECON_PRESET_NONE) return 1;
    int da = move_dir(H, af, at), db = move_dir(H, bf, bt);
    if (da != db) return 0;
    if (da <= 1) return af / H == bf / H;
    return af % H == bf % H;
}

static int dag_acyclic(int P, int64_t ne, const int32_t *es, const int32_t *ed) {
    int *indeg = xcalloc((size_t)P + 1, sizeof(int));
    int64_t *off = xcalloc((size_t)P + 2, 8);
    int32_t *adj = xcalloc((size_t)ne + 1, 4);
    for (int64_t e = 0; e < ne; ++e) {
        if (es[e] < 0 || es[e] >= P || ed[e] < 0 || ed[e] >= P) {
            free(indeg);
            free(off);
            free(adj);
            return 0;
        }
        ++off[es[e] + 1];
        ++indeg[ed[e]];
    }
    for (int i = 0; i < P; ++i) off[i + 1] += off[i];
    int64_t *fill = xcalloc((size_t)P + 1, 8);
    for (int64_t e = 0; e < ne; ++e) adj[off[es[e]] + fill[es[e]]++] = ed[e];
    int *stack = xcalloc((size_t)P + 1, sizeof(int));
    int top = 0, seen = 0;
    for (int i = 0; i < P; ++i)
        if (!indeg[i]) stack[top++] = i;
    while (top) {
        int i = stack[--top];
        ++seen;
        for (int64_t q = off[i]; q < off[i + 1]; ++q)
            if (--indeg[adj[q]] == 0) stack[top++] = adj[q];
    }
    free(indeg);
    free(off);
    free(adj);
    free(fill);
    free(stack);
    return seen == P;
}

static recon_status batch_core(int W, int H, const uint64_t *occ, int P, const int64_t *off,
                               const int32_t *verts, int64_t ne, const int32_t *es, const int32_t *ed,
                               int preset, int edge_level, int32_t *move_batch, int64_t *nbatches,
                               int32_t *detail) {
    *detail = 0;
    *nbatches = 0;
    if (!dag_acyclic(P, ne, es, ed)) {
        *detail = RECON_D_BATCH_CYCLIC;
        return RECON_ERR_INPUT;
    }
    const int64_t N = (int64_t)W * H;
    char *occv = xcalloc((size_t)N, 1), *inb = xcalloc((size_t)N, 1);
    const int wpc = wpc_of(H);
    for (int x = 0; x < W; ++x)
        for (int y = 0; y < H; ++y)
            if ((occ[(size_t)x * wpc + y / 64] >> (y % 64)) & 1ULL) occv[x * H + y] = 1;
    int64_t *soff = xcalloc((size_t)P + 2, 8);
    int32_t *succ = xcalloc((size_t)ne + 1, 4);
    int *blockers = xcalloc((size_t)P + 1, sizeof(int));
    for (int64_t e = 0; e < ne; ++e) {
        ++soff[es[e] + 1];
        ++blockers[ed[e]];
    }
    for (int i = 0; i < P; ++i) soff[i + 1] += soff[i];
    int64_t *fill = xcalloc((size_t)P + 1, 8);
    for (int64_t e = 0; e < ne; ++e) succ[soff[es[e]] + fill[es[e]]++] = ed[e];
    /* edge-level release thresholds (batching.cpp:38-59) */
    int64_t *need = NULL;
    if (edge_level) {
        need = xcalloc((size_t)ne + 1, 8);
        char *touched = xcalloc((size_t)N, 1);
        for (int64_t e = 0; e < ne; ++e) {
            int i = es[e], j = ed[e];
            for (int64_t q = off[j]; q < off[j + 1]; ++q) touched[verts[q]] = 1;
            int64_t nd = 0, li = off[i + 1] - off[i] - 1;
            for (int64_t k = 0; k < li; ++k)
                if (touched[verts[off[i] + k]] || touched[verts[off[i] + k + 1]]) nd = k + 1;
            for (int64_t q = off[j]; q < off[j + 1]; ++q) touched[verts[q]] = 0;
            need[e] = nd;
        }
        free(touched);
    }
    int64_t *next = xcalloc((size_t)P + 1, 8);
    char *done = xcalloc((size_t)P + 1, 1), *ready = xcalloc((size_t)P + 1, 1);
    int *newly = xcalloc((size_t)P + 1, sizeof(int));
    int nnew = 0;
    int64_t total_left = 0;
#define FINISH(pid)                                                  \
    do {                                                             \
        done[pid] = 1;                                               \
        for (int64_t q_ = soff[pid]; q_ < soff[(pid) + 1]; ++q_)     \
            if (--blockers[succ[q_]] == 0) newly[nnew++] = succ[q_]; \
    } while (0)
    for (int i = 0; i < P; ++i) {
        int64_t len = off[i + 1] - off[i] - 1;
        total_left += len;
        if (len == 0) FINISH(i);
    }
    for (int i = 0; i < P; ++i)
        if (!done[i] && blockers[i] == 0) ready[i] = 1;
    nnew = 0;
    int32_t *queue = xcalloc((size_t)P + 1, 4), *members = xcalloc((size_t)P + 1, 4);
    int32_t *mf = xcalloc((size_t)P + 1, 4), *mt = xcalloc((size_t)P + 1, 4);
    recon_status st = RECON_OK;
    int64_t nb = 0;
    while (total_left > 0) {
        int nq = 0, nm = 0;
        if (edge_level) {
            for (int i = 0; i < P; ++i) {
                if (done[i]) continue;
                int ok = 1;
                for (int64_t e = 0; e < ne && ok; ++e)
                    if (ed[e] == i && !done[es[e]] && next[es[e]] < need[e]) ok = 0;
                if (ok) queue[nq++] = i;
            }
        } else {
            for (int i = 0; i < P; ++i)
                if (ready[i]) queue[nq++] = i;
        }
        for (int q = 0; q < nq; ++q) {
            int pid = queue[q];
            int32_t f = verts[off[pid] + next[pid]], t = verts[off[pid] + next[pid] + 1];
            if (occv[t]) continue;
            if (inb[f] || inb[t]) continue;
            int ok = 1;
            for (int m = 0; m < nm && ok; ++m) ok = compatible(preset, H, f, t, mf[m], mt[m]);
            if (!ok) continue;
            mf[nm] = f;
            mt[nm] = t;
            members[nm++] = pid;
            inb[f] = inb[t] = 1;
        }
        if (nm == 0) {
            *detail = RECON_D_BATCH_NO_PROGRESS;
            st = RECON_ERR_INPUT;
            break;
        }
        for (int m = 0; m < nm; ++m) {
            occv[mf[m]] = 0;
            inb[mf[m]] = inb[mt[m]] = 0;
        }
        for (int m = 0; m < nm; ++m) occv[mt[m]] = 1;
        for (int m = 0; m < nm; ++m) {
            int pid = members[m];
            move_batch[off[pid] - pid + next[pid]] = (int32_t)nb;
            ++next[pid];
            --total_left;
            if (next[pid] == off[pid + 1] - off[pid] - 1) {
                ready[pid] = 0;
                FINISH(pid);
            }
        }
        for (int q = 0; q < nnew; ++q) ready[newly[q]] = 1;
        nnew = 0;
        ++nb;
    }
#undef FINISH
    *nbatches = st == RECON_OK ? nb : 0;
    free(occv);
    free(inb);
    free(soff);
    free(succ);
    free(blockers);
    free(fill);
    free(need);
    free(next);
    free(done);
    free(ready);
    free(newly);
    free(queue);
    free(members);
    free(mf);
    free(mt);
    return st;
}

recon_status recon_batch_moves(recon_ctx *ctx, int32_t width, int32_t height, const uint64_t *occ,
                               int32_t path_count, const int64_t *path_offsets,
                               const int32_t *path_vertices, int64_t edge_count,
                               const int32_t *edge_src, const int32_t *edge_dst, int32_t preset,
                               int32_t edge_level, int32_t *move_batch, int64_t *batch_count,
                               int32_t *detail) {
    (void)ctx;
    int32_t det = 0;
    recon_status st = batch_core(width, height, occ, path_count, path_offsets, path_vertices, edge_count,
                                 edge_src, edge_dst, preset, edge_level, move_batch, batch_count, &det);
    if (detail) *detail = det;
    return st;
}

recon_status recon_pipeline_batch_run(recon_ctx *ctx, const recon_pipeline_batch *pb) {
    (void)ctx;
    const recon_grid_batch *b = &pb->grid;
    const int W = b->width, H = b->height, wpc = wpc_of(H);
    const int64_t stride = (int64_t)W * b->h_prime;
    for (int i = 0; i < b->count; ++i) {
        recon_grid_solution out;
        memset(&out, 0, sizeof(out));
        out.path_src = b->path_src + i * stride;
        out.path_dst = b->path_dst + i * stride;
        out.path_event = b->path_event ? b->path_event + i * stride : NULL;
        out.path_capacity = stride;
        int32_t det = 0;
        const uint64_t *occ = b->occ + (size_t)i * W * wpc;
        recon_status st = grid_solve(pb->solver == 1, occ, W, H, b->h_prime, &out, &det);
        int64_t nb = 0;
        if (st == RECON_OK) {
            int64_t P = out.path_count;
            int64_t *off = xcalloc((size_t)P + 2, 8);
            int32_t *verts = xcalloc((size_t)(out.total_displacement + P + 1), 4);
            for (int64_t p = 0; p < P; ++p)
                off[p + 1] = off[p] + walk_path(H, out.path_src[p], out.path_dst[p], verts + off[p]);
            edge_t *e = NULL;
            int64_t ne = dag_edges(W, H, out.path_src, out.path_dst, P, &e);
            int32_t *es = xcalloc((size_t)ne + 1, 4), *ed = xcalloc((size_t)ne + 1, 4);
            for (int64_t q = 0; q < ne; ++q) {
                es[q] = e[q].a;
                ed[q] = e[q].b;
            }
            if (out.total_displacement > pb->move_stride) st = RECON_ERR_CAPACITY;
            else
                st = batch_core(W, H, occ, (int)P, off, verts, ne, es, ed, pb->preset, 0,
                                pb->move_batch + i * pb->move_stride, &nb, &det);
            free(off);
            free(verts);
            free(e);
            free(es);
            free(ed);
        }
        b->status[i] = st;
        if (b->detail) b->detail[i] = det;
        b->path_count[i] = (int32_t)out.path_count;
        b->total_displacement[i] = out.total_displacement;
        pb->batch_count[i] = (int32_t)nb;
    }
    return RECON_OK;
}

recon_status recon_pipeline_batch_run_host(recon_ctx *ctx, const recon_pipeline_batch *pb) {
    return recon_pipeline_batch_run(ctx, pb);
}

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return x < y ? -1 : (x > y);
}

/* min_assignment_cost_1d (exact1d.cpp:320-326): window DP over grouped sources */
recon_status recon_min_cost_1d(recon_ctx *ctx, int32_t ns, const int64_t *sources, int32_t nt, const int64_t *targets,
                               int64_t *cost, int32_t *detail) {
    (void)ctx;
    if (detail) *detail = 0;
    *cost = 0;
    if (nt == 0) return RECON_OK;
    if (ns < nt) {
        if (detail) *detail = RECON_D_INFEASIBLE_SUPPLY;
        return RECON_ERR_INFEASIBLE;
    }
    int64_t *s = xcalloc((size_t)ns, 8), *t = xcalloc((size_t)nt, 8), *pos = xcalloc((size_t)ns, 8);
    int32_t *lo = xcalloc((size_t)ns, 4), *hi = xcalloc((size_t)ns, 4), *use = xcalloc((size_t)ns, 4);
    memcpy(s, sources, (size_t)ns * 8);
    memcpy(t, targets, (size_t)nt * 8);
    qsort(s, (size_t)ns, 8, cmp_i64);
    qsort(t, (size_t)nt, 8, cmp_i64);
    int np = 0;
    for (int i = 0; i < ns; ++i) {
        if (np && pos[np - 1] == s[i]) ++hi[np - 1];
        else {
            pos[np] = s[i];
            hi[np] = 1;
            ++np;
        }
    }
    window_dp(np, pos, lo, hi, nt, t, use, cost);
    free(s);
    free(t);
    free(pos);
    free(lo);
    free(hi);
    free(use);
    return RECON_OK;
}

recon_status recon_occupancy_dag_paths(recon_ctx *ctx, int32_t width, int32_t height, int32_t P, const int64_t *off,
                                       const int32_t *verts, int32_t *dag_src, int32_t *dag_dst, int64_t dag_capacity,
                                       int64_t *dag_count, int32_t *detail) {
    (void)ctx;
    if (detail) *detail = 0;
    int64_t N = (int64_t)width * height;
    int32_t *so = xcalloc((size_t)N, 4), *to = xcalloc((size_t)N, 4);
    for (int64_t v = 0; v < N; ++v) so[v] = to[v] = -1;
    for (int i = 0; i < P; ++i) {
        so[verts[off[i]]] = i;
        to[verts[off[i + 1] - 1]] = i;
    }
    int64_t cap = 64, ne = 0;
    edge_t *e = xcalloc((size_t)cap, sizeof(edge_t));
    for (int i = 0; i < P; ++i)
        for (int64_t q = off[i]; q < off[i + 1]; ++q) {
            int32_t v = verts[q];
            if (ne + 2 > cap) {
                cap *= 2;
                e = realloc(e, (size_t)cap * sizeof(edge_t));
            }
            if (so[v] >= 0 && so[v] != i) e[ne++] = (edge_t){so[v], i};
            if (to[v] >= 0 && to[v] != i) e[ne++] = (edge_t){i, to[v]};
        }
    qsort(e, (size_t)ne, sizeof(edge_t), cmp_edge);
    int64_t u = 0;
    for (int64_t i = 0; i < ne; ++i)
        if (u == 0 || e[i].a != e[u - 1].a || e[i].b != e[u - 1].b) e[u++] = e[i];
    *dag_count = u;
    recon_status st = RECON_OK;
    if (u > dag_capacity) st = RECON_ERR_CAPACITY;
    else
        for (int64_t i = 0; i < u; ++i) {
            dag_src[i] = e[i].a;
            dag_dst[i] = e[i].b;
        }
    free(so);
    free(to);
    free(e);
    return st;
}

/* ======================================================================== */
/* Validators: sequential restatement of validate_solution                  */
/* (executor.cpp:142-183), check_one_move_per_token (executor.cpp:185-219)  */
/* and validate_batches (batching.cpp:161-252) for one-bend grid solutions  */
/* with the identity schedule.                                               */
/* ======================================================================== */

/* Kahn's algorithm (MoveDag::topo_order, path_system.cpp) */
static int edges_acyclic(int64_t np, const edge_t *e, int64_t ne) {
    int32_t *indeg = xcalloc((size_t)np, 4), *q = xcalloc((size_t)np, 4);
    int64_t *off = xcalloc((size_t)np + 1, 8);
    int32_t *adj = xcalloc((size_t)ne, 4);
    for (int64_t i = 0; i < ne; ++i) {
        off[e[i].a + 1]++;
        indeg[e[i].b]++;
    }
    for (int64_t i = 0; i < np; ++i) off[i + 1] += off[i];
    int64_t *cur = xcalloc((size_t)np + 1, 8);
    memcpy(cur, off, (size_t)(np + 1) * 8);
    for (int64_t i = 0; i < ne; ++i) adj[cur[e[i].a]++] = e[i].b;
    int64_t h = 0, t = 0;
    for (int64_t i = 0; i < np; ++i)
        if (!indeg[i]) q[t++] = (int32_t)i;
    while (h < t) {
        const int32_t u = q[h++];
        for (int64_t k = off[u]; k < off[u + 1]; ++k)
            if (--indeg[adj[k]] == 0) q[t++] = adj[k];
    }
    free(indeg);
    free(q);
    free(off);
    free(adj);
    free(cur);
    return t == np;
}

static uint32_t validate_one(int W, int H, int hp, const uint64_t *occ, const int32_t *ps, const int32_t *pt,
                             int64_t np, const int64_t *tdisp, const int32_t *displaced, int dag_mode,
                             const int32_t *ea, const int32_t *eb, int64_t ne_in, const int32_t *mb, int64_t nb,
                             int preset) {
    const int64_t V = (int64_t)W * H;
    const int wpc = wpc_of(H), ylo = (H - hp) / 2;
    uint32_t v = 0;
    char *seen_s = xcalloc((size_t)V, 1), *seen_t = xcalloc((size_t)V, 1), *ok = xcalloc((size_t)np, 1);
    int64_t *len = xcalloc((size_t)np, 8), *off = xcalloc((size_t)np + 1, 8);
    int64_t weight = 0, moved = 0;
    /* check_paths (executor.cpp:38-80) */
    for (int64_t i = 0; i < np; ++i) {
        if (ps[i] < 0 || ps[i] >= V || pt[i] < 0 || pt[i] >= V) {
            v |= RECON_V_PATH_BOUNDS;
            continue;
        }
        ok[i] = 1;
        const int dx = ps[i] / H - pt[i] / H, dy = ps[i] % H - pt[i] % H;
        len[i] = (dx < 0 ? -dx : dx) + (dy < 0 ? -dy : dy);
        if (seen_s[ps[i]]) v |= RECON_V_SHARED_SOURCE;
        if (seen_t[pt[i]]) v |= RECON_V_SHARED_TARGET;
        seen_s[ps[i]] = seen_t[pt[i]] = 1;
    }
    if (v & RECON_V_PATH_BOUNDS) { /* endpoints off the grid: nothing else is evaluated */
        free(seen_s);
        free(seen_t);
        free(ok);
        free(len);
        free(off);
        return RECON_V_PATH_BOUNDS;
    }
    for (int64_t i = 0; i < np; ++i) {
        off[i + 1] = off[i] + len[i];
        weight += len[i];
        moved += len[i] > 0;
    }
    /* the dag */
    edge_t *e = NULL;
    int64_t ne = 0;
    if (dag_mode == RECON_DAG_EXPLICIT) {
        e = xcalloc((size_t)ne_in, sizeof(edge_t));
        for (int64_t i = 0; i < ne_in; ++i) e[i] = (edge_t){ea[i], eb[i]};
        ne = ne_in;
    } else if (dag_mode == RECON_DAG_OCCUPANCY && !(v & RECON_V_PATH_BOUNDS)) {
        ne = dag_edges(W, H, ps, pt, np, &e);
    }
    if (ne && !edges_acyclic(np, e, ne)) v |= RECON_V_DAG_CYCLE;
    if (tdisp && *tdisp != weight) v |= RECON_V_STATS_DISPLACEMENT;
    if (displaced && *displaced != moved) v |= RECON_V_STATS_DISPLACED;
    int32_t *verts = xcalloc((size_t)(W + H + 2), 4);
    char *cfg = xcalloc((size_t)V, 1);
    if (!v) {
        for (int64_t x = 0; x < V; ++x) cfg[x] = getbit(occ + (x / H) * wpc, (int)(x % H));
        int fail = 0;
        for (int64_t i = 0; i < np && !fail; ++i) { /* execute_schedule (executor.cpp:10-26) */
            const int64_t nv = walk_path(H, ps[i], pt[i], verts);
            for (int64_t k = 0; k + 1 < nv && !fail; ++k) {
                if (!cfg[verts[k]] || cfg[verts[k + 1]]) fail = 1;
                cfg[verts[k]] = 0;
                cfg[verts[k + 1]] = 1;
            }
        }
        if (fail) {
            v |= RECON_V_EXECUTION;
        } else {
            for (int x = 0; x < W; ++x)
                for (int y = ylo; y < ylo + hp; ++y)
                    if (!cfg[(int64_t)x * H + y]) v |= RECON_V_TARGETS;
            for (int64_t k = 0; k < ne; ++k) { /* linear extension, identity schedule */
                const int32_t i = e[k].a, j = e[k].b;
                if (len[i] > 0 && len[j] > 0 && off[i] + len[i] - 1 > off[j]) {
                    v |= RECON_V_DAG_ORDER;
                    break;
                }
            }
        }
    }
    /* check_one_move_per_token (executor.cpp:185-219): match_schedule
       (executor.cpp:82-140, pending path fronts per vertex, first pending
       path whose next vertex fits) attributes each move to a path; then
       token identities are followed */
    {
        int32_t *head = xcalloc((size_t)V, 4), *tail = xcalloc((size_t)V, 4);
        int32_t *nx = xcalloc((size_t)np + 1, 4), *pv = xcalloc((size_t)np + 1, 4);
        int64_t *nextk = xcalloc((size_t)np + 1, 8);
        char *starts = xcalloc((size_t)weight + 1, 1);
        for (int64_t x = 0; x < V; ++x) head[x] = tail[x] = -1;
#define PUSH(vv, pid)                                   \
    do {                                                \
        nx[pid] = -1;                                   \
        pv[pid] = tail[vv];                             \
        if (tail[vv] >= 0) nx[tail[vv]] = (int32_t)(pid); \
        else head[vv] = (int32_t)(pid);                  \
        tail[vv] = (int32_t)(pid);                       \
    } while (0)
        for (int64_t i = 0; i < np; ++i)
            if (len[i] > 0) PUSH(ps[i], i);
        int matched_all = 1;
        int64_t mi = 0;
        int32_t *pv2 = xcalloc((size_t)(W + H + 2), 4);
        for (int64_t i = 0; i < np && matched_all; ++i) {
            const int64_t nv = walk_path(H, ps[i], pt[i], verts);
            for (int64_t k = 0; k + 1 < nv; ++k, ++mi) {
                const int32_t from = verts[k], to = verts[k + 1];
                int32_t m = -1;
                for (int32_t q = head[from]; q >= 0; q = nx[q]) {
                    walk_path(H, ps[q], pt[q], pv2);
                    if (pv2[nextk[q] + 1] == to) {
                        m = q;
                        break;
                    }
                }
                if (m < 0) {
                    matched_all = 0;
                    break;
                }
                if (pv[m] >= 0) nx[pv[m]] = nx[m];
                else head[from] = nx[m];
                if (nx[m] >= 0) pv[nx[m]] = pv[m];
                else tail[from] = pv[m];
                starts[mi] = nextk[m] == 0;
                const int64_t kk = ++nextk[m];
                if (kk < len[m]) {
                    walk_path(H, ps[m], pt[m], pv2);
                    PUSH(pv2[kk], m);
                }
            }
        }
#undef PUSH
        if (!matched_all) {
            v |= RECON_V_TOKEN_MATCH;
        } else {
            int32_t *tok = xcalloc((size_t)V, 4);
            for (int64_t x = 0; x < V; ++x) tok[x] = getbit(occ + (x / H) * wpc, (int)(x % H)) ? (int32_t)x : -1;
            char *began = xcalloc((size_t)V, 1);
            int stop = 0;
            mi = 0;
            for (int64_t i = 0; i < np && !stop; ++i) {
                const int64_t nv = walk_path(H, ps[i], pt[i], verts);
                for (int64_t k = 0; k + 1 < nv; ++k, ++mi) {
                    const int32_t t = tok[verts[k]];
                    if (t < 0) {
                        v |= RECON_V_TOKEN_EMPTY;
                        stop = 1;
                        break;
                    }
                    if (starts[mi]) {
                        if (began[t]) {
                            v |= RECON_V_TOKEN_SECOND_PATH;
                            stop = 1;
                            break;
                        }
                        began[t] = 1;
                    }
                    tok[verts[k]] = -1;
                    tok[verts[k + 1]] = t;
                }
            }
            free(tok);
            free(began);
        }
        free(head);
        free(tail);
        free(nx);
        free(pv);
        free(nextk);
        free(starts);
        free(pv2);
    }
    /* validate_batches (batching.cpp:161-252) */
    if (mb) {
        uint32_t bv = 0;
        int64_t *bcnt = xcalloc((size_t)nb + 1, 8), *bstart = xcalloc((size_t)nb + 2, 8);
        for (int64_t i = 0; i < np; ++i)
            for (int64_t k = 0; k < len[i]; ++k) {
                const int32_t b = mb[off[i] + k];
                if (b < 0 || b >= nb) bv |= RECON_V_BATCH_CONSERVATION;
                else bcnt[b]++;
            }
        if (nb > weight) bv |= RECON_V_BATCH_BOUND;
        for (int64_t b = 0; b < nb; ++b) bstart[b + 1] = bstart[b] + bcnt[b];
        int32_t *mf = xcalloc((size_t)bstart[nb] + 1, 4), *mt = xcalloc((size_t)bstart[nb] + 1, 4);
        int64_t *fill = xcalloc((size_t)nb + 1, 8);
        for (int64_t i = 0; i < np; ++i) { /* batch b = its moves in ascending path id */
            if (!ok[i]) continue;
            const int64_t nv = walk_path(H, ps[i], pt[i], verts);
            for (int64_t k = 0; k + 1 < nv; ++k) {
                const int32_t b = mb[off[i] + k];
                if (b < 0 || b >= nb) continue;
                const int64_t at = bstart[b] + fill[b]++;
                mf[at] = verts[k];
                mt[at] = verts[k + 1];
            }
        }
        for (int64_t x = 0; x < V; ++x) cfg[x] = getbit(occ + (x / H) * wpc, (int)(x % H));
        char *used = xcalloc((size_t)V, 1);
        int ret = 0;
        for (int64_t b = 0; b < nb && !ret; ++b) {
            const int64_t s = bstart[b], n = bcnt[b];
            if (!n) {
                bv |= RECON_V_BATCH_EMPTY;
                continue;
            }
            for (int64_t m = s; m < s + n; ++m) {
                if (used[mf[m]] || used[mt[m]]) {
                    bv |= RECON_V_BATCH_DISJOINT;
                    ret = 1;
                    break;
                }
                used[mf[m]] = used[mt[m]] = 1;
            }
            for (int64_t m = s; m < s + n; ++m) used[mf[m]] = used[mt[m]] = 0;
            if (ret) break;
            if (preset == RECON_PRESET_COLUMN_DIRECTION) { /* ConstraintSet::compatible (batching.cpp:17-24) */
                int bad = 0;
                for (int64_t m = s + 1; m < s + n && !bad; ++m) {
                    const int fx0 = mf[s] / H, fy0 = mf[s] % H, tx0 = mt[s] / H, ty0 = mt[s] % H;
                    const int fx = mf[m] / H, fy = mf[m] % H, tx = mt[m] / H, ty = mt[m] % H;
                    const int d0 = ty0 > fy0 ? 0 : ty0 < fy0 ? 1 : tx0 < fx0 ? 2 : 3;
                    const int d = ty > fy ? 0 : ty < fy ? 1 : tx < fx ? 2 : 3;
                    if (d != d0 || (d < 2 ? fx != fx0 : fy != fy0)) bad = 1;
                }
                if (bad) bv |= RECON_V_BATCH_CONSTRAINT;
            }
            for (int64_t m = s; m < s + n; ++m)
                if (!cfg[mf[m]] || cfg[mt[m]]) {
                    bv |= RECON_V_BATCH_COLLISION;
                    ret = 1;
                    break;
                }
            if (ret) break;
            for (int64_t m = s; m < s + n; ++m) cfg[mf[m]] = 0;
            for (int64_t m = s; m < s + n; ++m) cfg[mt[m]] = 1;
        }
        if (!ret) {
            for (int x = 0; x < W; ++x)
                for (int y = ylo; y < ylo + hp; ++y)
                    if (!cfg[(int64_t)x * H + y]) bv |= RECON_V_BATCH_TARGETS;
            if (!bv) {
                /* match_schedule on the batch-ordered move list: a path's moves
                   must appear in batch order; then dag order by first moves */
                for (int64_t i = 0; i < np && !bv; ++i)
                    for (int64_t k = 1; k < len[i]; ++k)
                        if (mb[off[i] + k] < mb[off[i] + k - 1]) {
                            bv |= RECON_V_BATCH_ORDER;
                            break;
                        }
                for (int64_t k = 0; k < ne && !bv; ++k) {
                    const int32_t i = e[k].a, j = e[k].b;
                    if (len[i] > 0 && len[j] > 0 && mb[off[j]] < mb[off[i]]) bv |= RECON_V_BATCH_DAG;
                }
            }
        }
        v |= bv;
        free(bcnt);
        free(bstart);
        free(mf);
        free(mt);
        free(fill);
        free(used);
    }
    free(seen_s);
    free(seen_t);
    free(ok);
    free(len);
    free(off);
    free(e);
    free(verts);
    free(cfg);
    return v;
}

static recon_status validate_run(const recon_validate_batch *b) {
    if (!b || !b->occ || !b->path_src || !b->path_dst || !b->path_count || !b->verdict) return RECON_ERR_ARGUMENT;
    const int wpc = wpc_of(b->height);
    for (int32_t i = 0; i < b->count; ++i) {
        const int64_t e0 = b->dag_mode == RECON_DAG_EXPLICIT ? b->dag_offset[i] : 0;
        const int64_t e1 = b->dag_mode == RECON_DAG_EXPLICIT ? b->dag_offset[i + 1] : 0;
        b->verdict[i] = validate_one(
            b->width, b->height, b->h_prime, b->occ + (size_t)i * b->width * wpc, b->path_src + i * b->path_stride,
            b->path_dst + i * b->path_stride, b->path_count[i], b->total_displacement ? b->total_displacement + i : NULL,
            b->displaced ? b->displaced + i : NULL, b->dag_mode, b->dag_a ? b->dag_a + e0 : NULL,
            b->dag_b ? b->dag_b + e0 : NULL, e1 - e0, b->move_batch ? b->move_batch + i * b->move_stride : NULL,
            b->batch_count ? b->batch_count[i] : 0, b->preset);
    }
    return RECON_OK;
}

recon_status recon_validate_batch_run(recon_ctx *c, const recon_validate_batch *b) {
    (void)c;
    return validate_run(b);
}
recon_status recon_validate_batch_run_host(recon_ctx *c, const recon_validate_batch *b) {
    (void)c;
    return validate_run(b);
}

/* ======================================================================== */
/* Wire formats: solution_to_json / batch_schedule_to_json (io.cpp:81-164)  */
/* in the stock nlohmann dump(2) layout                                      */
/* ======================================================================== */

typedef struct {
    char *p;
    int64_t n, cap;
} sbuf;

static void sb_put(sbuf *b, const char *s, int64_t n) {
    if (b->n + n > b->cap) {
        while (b->n + n > b->cap) b->cap = b->cap ? 2 * b->cap : 4096;
        b->p = realloc(b->p, (size_t)b->cap);
    }
    memcpy(b->p + b->n, s, (size_t)n);
    b->n += n;
}
static void sb_str(sbuf *b, const char *s) { sb_put(b, s, (int64_t)strlen(s)); }
static void sb_sp(sbuf *b, int k) {
    for (int i = 0; i < k; ++i) sb_put(b, " ", 1);
}
static void sb_num(sbuf *b, long long v) {
    char t[32];
    int n = snprintf(t, sizeof t, "%lld", v);
    sb_put(b, t, n);
}
static void sb_xy(sbuf *b, int ind, int H, int v) { /* caller wrote the indent */
    sb_str(b, "[\n");
    sb_sp(b, ind + 2);
    sb_num(b, v / H);
    sb_str(b, ",\n");
    sb_sp(b, ind + 2);
    sb_num(b, v % H);
    sb_str(b, "\n");
    sb_sp(b, ind);
    sb_str(b, "]");
}
static void sb_move(sbuf *b, int ind, int H, int from, int to) {
    sb_sp(b, ind);
    sb_str(b, "[\n");
    sb_sp(b, ind + 2);
    sb_xy(b, ind + 2, H, from);
    sb_str(b, ",\n");
    sb_sp(b, ind + 2);
    sb_xy(b, ind + 2, H, to);
    sb_str(b, "\n");
    sb_sp(b, ind);
    sb_str(b, "]");
}

static recon_status sb_finish(sbuf *b, char *out, int64_t cap, int64_t *length) {
    *length = b->n;
    recon_status st = RECON_OK;
    if (cap < b->n) st = RECON_ERR_CAPACITY;
    else if (b->n) memcpy(out, b->p, (size_t)b->n);
    free(b->p);
    return st;
}

static recon_status oracle_solution_json(int32_t width, int32_t H, int32_t np, const int32_t *ps, const int32_t *pt,
                                         const int32_t *order, int64_t ne, const int32_t *ea, const int32_t *eb,
                                         int64_t displaced, int64_t total, char *out, int64_t cap, int64_t *length) {
    sbuf b = {0};
    int32_t *verts = xcalloc((size_t)(width + H + 2), 4);
    sb_str(&b, "{\n  \"moves\": ");
    int first = 1;
    for (int32_t i = 0; i < np; ++i) {
        const int32_t q = order ? order[i] : i;
        const int64_t nv = walk_path(H, ps[q], pt[q], verts);
        for (int64_t k = 0; k + 1 < nv; ++k) {
            sb_str(&b, first ? "[\n" : ",\n");
            first = 0;
            sb_move(&b, 4, H, verts[k], verts[k + 1]);
        }
    }
    sb_str(&b, first ? "[],\n" : "\n  ],\n");
    sb_str(&b, "  \"dag_edges\": ");
    for (int64_t e = 0; e < ne; ++e) {
        sb_str(&b, e ? ",\n" : "[\n");
        sb_sp(&b, 4);
        sb_str(&b, "[\n");
        sb_sp(&b, 6);
        sb_num(&b, ea[e]);
        sb_str(&b, ",\n");
        sb_sp(&b, 6);
        sb_num(&b, eb[e]);
        sb_str(&b, "\n    ]");
    }
    sb_str(&b, ne ? "\n  ],\n" : "[],\n");
    sb_str(&b, "  \"paths\": ");
    for (int32_t q = 0; q < np; ++q) {
        sb_str(&b, q ? ",\n" : "[\n");
        sb_sp(&b, 4);
        sb_str(&b, "[\n");
        const int64_t nv = walk_path(H, ps[q], pt[q], verts);
        for (int64_t k = 0; k < nv; ++k) {
            if (k) sb_str(&b, ",\n");
            sb_sp(&b, 6);
            sb_xy(&b, 6, H, verts[k]);
        }
        sb_str(&b, "\n    ]");
    }
    sb_str(&b, np ? "\n  ],\n" : "[],\n");
    sb_str(&b, "  \"stats\": {\n    \"displaced_tokens\": ");
    sb_num(&b, displaced);
    sb_str(&b, ",\n    \"total_displacement\": ");
    sb_num(&b, total);
    sb_str(&b, "\n  }\n}\n");
    free(verts);
    return sb_finish(&b, out, cap, length);
}

static recon_status oracle_batch_json(int32_t width, int32_t H, int32_t np, const int32_t *ps, const int32_t *pt,
                                      const int32_t *mb, int32_t nb, int32_t preset, char *out, int64_t cap,
                                      int64_t *length) {
    sbuf b = {0};
    int32_t *verts = xcalloc((size_t)(width + H + 2), 4);
    int64_t D = 0;
    for (int32_t q = 0; q < np; ++q) {
        const int dx = ps[q] / H - pt[q] / H, dy = ps[q] % H - pt[q] % H;
        D += (dx < 0 ? -dx : dx) + (dy < 0 ? -dy : dy);
    }
    int64_t *cnt = xcalloc((size_t)nb + 1, 8), *st = xcalloc((size_t)nb + 2, 8), *fill = xcalloc((size_t)nb + 1, 8);
    int32_t *mf = xcalloc((size_t)D + 1, 4), *mt = xcalloc((size_t)D + 1, 4);
    for (int64_t m = 0; m < D; ++m)
        if (mb[m] >= 0 && mb[m] < nb) cnt[mb[m]]++;
    for (int32_t k = 0; k < nb; ++k) st[k + 1] = st[k] + cnt[k];
    int64_t m = 0;
    for (int32_t q = 0; q < np; ++q) {
        const int64_t nv = walk_path(H, ps[q], pt[q], verts);
        for (int64_t k = 0; k + 1 < nv; ++k, ++m) {
            const int32_t bi = mb[m];
            if (bi < 0 || bi >= nb) continue;
            mf[st[bi] + fill[bi]] = verts[k];
            mt[st[bi] + fill[bi]++] = verts[k + 1];
        }
    }
    sb_str(&b, "{\n  \"batches\": ");
    int any = 0;
    for (int32_t k = 0; k < nb; ++k) {
        if (!cnt[k]) continue; /* a schedule from batching has no empty batch */
        sb_str(&b, any ? ",\n" : "[\n");
        any = 1;
        const char *ax = "null", *dr = "null";
        if (preset == RECON_PRESET_COLUMN_DIRECTION) {
            const int f = mf[st[k]], t = mt[st[k]];
            const int fx = f / H, fy = f % H, tx = t / H, ty = t % H;
            if (ty > fy) ax = "\"col\"", dr = "\"up\"";
            else if (ty < fy) ax = "\"col\"", dr = "\"down\"";
            else if (tx < fx) ax = "\"row\"", dr = "\"left\"";
            else ax = "\"row\"", dr = "\"right\"";
        }
        sb_str(&b, "    {\n      \"axis\": ");
        sb_str(&b, ax);
        sb_str(&b, ",\n      \"dir\": ");
        sb_str(&b, dr);
        sb_str(&b, ",\n      \"moves\": [\n");
        for (int64_t x = st[k]; x < st[k + 1]; ++x) {
            if (x > st[k]) sb_str(&b, ",\n");
            sb_move(&b, 8, H, mf[x], mt[x]);
        }
        sb_str(&b, "\n      ]\n    }");
    }
    sb_str(&b, any ? "\n  ]\n}\n" : "[]\n}\n");
    free(verts);
    free(cnt);
    free(st);
    free(fill);
    free(mf);
    free(mt);
    return sb_finish(&b, out, cap, length);
}

recon_status recon_solution_json(recon_ctx *c, int32_t width, int32_t height, int32_t np, const int32_t *ps,
                                 const int32_t *pt, const int32_t *order, int64_t ne, const int32_t *ea,
                                 const int32_t *eb, int64_t displaced, int64_t total, char *out, int64_t cap,
                                 int64_t *length) {
    (void)c;
    if (!length || width <= 0 || height <= 0 || np < 0 || ne < 0) return RECON_ERR_ARGUMENT;
    return oracle_solution_json(width, height, np, ps, pt, order, ne, ea, eb, displaced, total, out, cap, length);
}
recon_status recon_solution_json_host(recon_ctx *c, int32_t width, int32_t height, int32_t np, const int32_t *ps,
                                      const int32_t *pt, const int32_t *order, int64_t ne, const int32_t *ea,
                                      const int32_t *eb, int64_t displaced, int64_t total, char *out, int64_t cap,
                                      int64_t *length) {
    return recon_solution_json(c, width, height, np, ps, pt, order, ne, ea, eb, displaced, total, out, cap, length);
}
recon_status recon_batch_schedule_json(recon_ctx *c, int32_t width, int32_t height, int32_t np, const int32_t *ps,
                                       const int32_t *pt, const int32_t *mb, int32_t nb, int32_t preset, char *out,
                                       int64_t cap, int64_t *length) {
    (void)c;
    if (!length || width <= 0 || height <= 0 || np < 0 || nb < 0) return RECON_ERR_ARGUMENT;
    return oracle_batch_json(width, height, np, ps, pt, mb, nb, preset, out, cap, length);
}
recon_status recon_batch_schedule_json_host(recon_ctx *c, int32_t width, int32_t height, int32_t np,
                                            const int32_t *ps, const int32_t *pt, const int32_t *mb, int32_t nb,
                                            int32_t preset, char *out, int64_t cap, int64_t *length) {
    return recon_batch_schedule_json(c, width, height, np, ps, pt, mb, nb, preset, out, cap, length);
}

/* ======================================================================== */
/* Loss simulation: oracle/sim_common.h with this library's own solvers     */
/* ======================================================================== */

static recon_status oracle_sim_solve(int batching, int solver, int preset, recon_grid_batch *g, int64_t ms,
                                     int32_t *mb, int32_t *nb) {
    if (batching) {
        recon_pipeline_batch pb = {*g, solver, preset, ms, mb, nb};
        return recon_pipeline_batch_run_host(NULL, &pb);
    }
    return solver == 1 ? recon_bird_solve_batch_host(NULL, g) : recon_redrec_solve_batch_host(NULL, g);
}

#include "sim_common.h"

recon_status recon_sim_run_host(recon_ctx *c, const recon_sim_batch *b) {
    (void)c;
    return sim_run_checked(b, oracle_sim_solve);
}

/* recon_pipeline_stats over host pointers (digest_cpu.h) */
recon_status recon_pipeline_stats(recon_ctx *ctx, const recon_pipeline_batch *pb, recon_instance_stats *stats) {
    (void)ctx;
    return recon_dg_stats(pb, stats);
}

/* no device phases on the CPU checker */
recon_status recon_ctx_phase_times(recon_ctx *ctx, float *ms, int32_t n) {
    (void)ctx;
    for (int32_t i = 0; ms && i < n; ++i) ms[i] = 0.0f;
    return RECON_OK;
}

recon_status recon_pipeline_schedule_runs(recon_ctx *ctx, const recon_pipeline_batch *pb, recon_schedule_runs *runs) {
    (void)ctx;
    return recon_dg_runs(pb, runs);
}

/* the pipeline into a temporary schedule, then its runs */
recon_status recon_pipeline_batch_run_host_runs(recon_ctx *ctx, const recon_pipeline_batch *pb,
                                                recon_schedule_runs *runs) {
    if (!pb || !runs) return RECON_ERR_ARGUMENT;
    recon_pipeline_batch q = *pb;
    int32_t *tmp = NULL;
    if (!q.move_batch) {
        tmp = (int32_t *)malloc((size_t)pb->grid.count * (size_t)pb->move_stride * sizeof(int32_t));
        if (!tmp) return RECON_ERR_CAPACITY;
        q.move_batch = tmp;
    }
    recon_status st = recon_pipeline_batch_run_host(ctx, &q);
    if (st == RECON_OK) st = recon_dg_runs(&q, runs);
    free(tmp);
    return st;
}
