// recon_shim.cpp — the reference-side binding of the B200 library.
//
// Implements, from scratch, every function the reference declares in its
// hot-path headers (proj/include/recon/{exact1d,virtual_line,redrec,bird,
// batching}.hpp, unchanged) so that the reference's own code and tests link
// against it instead of src/{exact1d,virtual_line,redrec,bird,batching}.cpp.
//
// The solvers and every per-instance kernel go through the C-ABI
// (include/recon_b200.h) to the sm_100a kernels:
//   red_rec            -> recon_redrec_solve          (redrec.cpp:205-232)
//   bird               -> recon_bird_solve            (bird.cpp:107-123)
//   occupancy_dag      -> recon_occupancy_dag[_paths] (virtual_line.cpp:241-268)
//   assign_1d          -> recon_assign_1d             (exact1d.cpp:342-372)
//   assign_1d_generalized -> recon_assign_1d_generalized (exact1d.cpp:374-407)
//   min_assignment_cost_1d -> recon_min_cost_1d       (exact1d.cpp:320-326)
//   solve_1d           -> recon_solve_1d              (exact1d.cpp:564-572)
//   batch_moves        -> recon_batch_moves           (batching.cpp:28-159)
// The shim rebuilds the reference's value types from the compact device
// output (one-bend path shapes, orientations, labels, schedule, DAG) and
// rethrows statuses as the reference's exception types with its messages.
// The introspection helpers the reference exposes (select_best_pair,
// build_*_instance, realize_event, order_moves_1d, ...) are plain host C++
// re-implementations of the same contracts; they are not on the solve path.

#include <algorithm>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "recon/batching.hpp"
#include "recon/bird.hpp"
#include "recon/exact1d.hpp"
#include "recon/executor.hpp"
#include "recon/redrec.hpp"
#include "recon/virtual_line.hpp"
#include "recon_b200.h"

namespace recon {

namespace {

[[noreturn]] void rethrow(recon_status st, int32_t detail) {
    const std::string msg = recon_detail_message(detail);
    switch (st) {
        case RECON_ERR_INPUT: throw InputError(msg);
        case RECON_ERR_INFEASIBLE: throw InfeasibleError(msg);
        case RECON_ERR_COLLISION: throw CollisionError(msg);
        case RECON_ERR_LOGIC: throw std::logic_error(msg);
        case RECON_ERR_CUDA: throw std::runtime_error(std::string("recon_b200: ") + recon_last_cuda_error());
        default: throw std::runtime_error("recon_b200: status " + std::to_string(static_cast<int>(st)));
    }
}

void check(recon_status st, int32_t detail) {
    if (st != RECON_OK) rethrow(st, detail);
}

std::vector<uint64_t> pack_grid(const Geometry &g, const Configuration &c) {
    const int wpc = (g.height + 63) / 64;
    std::vector<uint64_t> occ(static_cast<size_t>(g.width) * wpc, 0ull);
    for (Vertex v : c.vertices()) {
        const Vec2 p = g.coords(v);
        occ[static_cast<size_t>(p.x) * wpc + p.y / 64] |= 1ull << (p.y % 64);
    }
    return occ;
}

std::vector<Vertex> staircase(const Geometry &g, Vertex s, Vertex t) {
    std::vector<Vertex> out;
    for (const Vec2 &v : shortest_path(g.coords(s), g.coords(t), StepPolicy::horizontal_first)) out.push_back(g.id(v));
    return out;
}

bool is_one_bend(const Geometry &g, const Path &p) {
    if (p.vertices.empty()) return false;
    return p.vertices == staircase(g, p.source(), p.target());
}

// Grid solution from the device's compact output: one-bend paths in canonical
// order, labels, orientation relative to the receiver's virtual line
// (virtual_line.cpp:150-173), identity schedule, occupancy DAG.
Solution grid_solution(const Geometry &g, BandSpec band, const std::vector<int32_t> &src,
                       const std::vector<int32_t> &dst, const std::vector<int32_t> &ev,
                       const std::vector<int32_t> &dag_a, const std::vector<int32_t> &dag_b) {
    PathSystem ps;
    ps.paths.reserve(src.size());
    for (size_t i = 0; i < src.size(); ++i) {
        Path p;
        p.vertices = staircase(g, src[i], dst[i]);
        const Vec2 a = g.coords(src[i]), b = g.coords(dst[i]);
        const int depth = g.row_from_top(a.y), dist = std::abs(a.x - b.x);
        const long long vpos = dist == 0 ? depth : (depth < band.lo ? depth - dist : depth + dist);
        p.orientation = g.row_from_top(b.y) > vpos ? Orientation::right : Orientation::left;
        p.event_id = ev[i];
        p.src_column = a.x;
        p.dst_column = b.x;
        ps.paths.push_back(std::move(p));
    }
    MoveDag dag;
    dag.node_count = static_cast<int>(ps.paths.size());
    for (size_t i = 0; i < dag_a.size(); ++i) dag.add_edge(dag_a[i], dag_b[i]);
    std::vector<int> order(ps.paths.size());
    std::iota(order.begin(), order.end(), 0);
    return make_solution(std::move(ps), std::move(dag), order);
}

template <typename Fn>
Solution run_grid(const Problem &problem, Fn solve, std::vector<int32_t> &events, int per_event) {
    const BandSpec band = derive_centered_band(problem);
    const Geometry &g = problem.geometry;
    const std::vector<uint64_t> occ = pack_grid(g, problem.sources);
    const int k = band.h_prime();
    std::vector<int32_t> src(static_cast<size_t>(g.width) * k), dst(src.size()), ev(src.size());
    events.assign(static_cast<size_t>(g.width) * per_event, 0);
    int64_t dag_cap = 4 * static_cast<int64_t>(src.size()) + 64;
    for (;;) {
        std::vector<int32_t> da(static_cast<size_t>(dag_cap)), db(static_cast<size_t>(dag_cap));
        recon_grid_solution out{};
        out.path_src = src.data();
        out.path_dst = dst.data();
        out.path_event = ev.data();
        out.path_capacity = static_cast<int64_t>(src.size());
        out.events = events.data();
        out.event_capacity = static_cast<int32_t>(events.size());
        out.dag_src = da.data();
        out.dag_dst = db.data();
        out.dag_capacity = dag_cap;
        int32_t detail = 0;
        const recon_status st = solve(occ.data(), g.width, g.height, k, &out, &detail);
        if (st == RECON_ERR_CAPACITY && out.dag_count > dag_cap) {
            dag_cap = out.dag_count;
            continue;
        }
        check(st, detail);
        src.resize(static_cast<size_t>(out.path_count));
        dst.resize(src.size());
        ev.resize(src.size());
        da.resize(static_cast<size_t>(out.dag_count));
        db.resize(da.size());
        events.resize(static_cast<size_t>(out.event_count) * per_event);
        return grid_solution(g, band, src, dst, ev, da, db);
    }
}

long long vpos_of(const VirtualToken &t) {
    if (t.dist == 0) return t.depth;
    return t.top_side ? t.depth - t.dist : t.depth + t.dist;
}

}  // namespace

// ===========================================================================
// exact1d.hpp
// ===========================================================================

Matching1D assign_1d(int n, std::vector<int> S, std::vector<int> T) {
    Matching1D m;
    std::vector<int64_t> ps(T.size() + 1), pt(T.size() + 1);
    m.use_count.assign(S.size(), 0);
    std::vector<int32_t> use(S.size() + 1);
    int64_t w = 0;
    int32_t detail = 0;
    check(recon_assign_1d(nullptr, n, S.data(), static_cast<int32_t>(S.size()), T.data(),
                          static_cast<int32_t>(T.size()), &w, ps.data(), pt.data(), use.data(), &detail),
          detail);
    m.weight = w;
    for (size_t i = 0; i < T.size(); ++i) m.pairs.emplace_back(ps[i], pt[i]);
    for (size_t i = 0; i < S.size(); ++i) m.use_count[i] = use[i];
    return m;
}

Matching1D assign_1d_generalized(const Generalized1DInstance &inst) {
    const size_t ns = inst.sources.size(), nt = inst.targets.size();
    std::vector<int64_t> pos(ns + 1), ps(nt + 1), pt(nt + 1);
    std::vector<int32_t> mult(ns + 1), mn(ns + 1), use(ns + 1);
    std::vector<int64_t> tg(inst.targets.begin(), inst.targets.end());
    tg.push_back(0);
    for (size_t i = 0; i < ns; ++i) {
        pos[i] = inst.sources[i].pos;
        mult[i] = inst.sources[i].multiplicity;
        mn[i] = inst.sources[i].min_use;
    }
    int64_t w = 0;
    int32_t detail = 0;
    check(recon_assign_1d_generalized(nullptr, static_cast<int32_t>(ns), pos.data(), mult.data(), mn.data(),
                                      static_cast<int32_t>(nt), tg.data(), &w, ps.data(), pt.data(),
                                      use.data(), &detail),
          detail);
    Matching1D m;
    m.weight = w;
    for (size_t i = 0; i < nt; ++i) m.pairs.emplace_back(ps[i], pt[i]);
    m.use_count.assign(use.begin(), use.begin() + static_cast<long>(ns));
    return m;
}

std::vector<int> level_vector(int n, const std::vector<int> &S, const std::vector<int> &T) {
    std::vector<int> s_at(static_cast<size_t>(n), 0), t_at(static_cast<size_t>(n), 0), out(static_cast<size_t>(n));
    for (int v : S) s_at[static_cast<size_t>(v)] = 1;
    for (int v : T) t_at[static_cast<size_t>(v)] = 1;
    int sp = 0, tp = 0;
    for (int i = 0; i < n; ++i) {
        sp += s_at[static_cast<size_t>(i)];
        out[static_cast<size_t>(i)] = sp - tp;  // targets counted strictly before i
        tp += t_at[static_cast<size_t>(i)];
    }
    return out;
}

long long min_assignment_cost_1d(const std::vector<long long> &sources, const std::vector<long long> &targets) {
    int64_t cost = 0;
    int32_t detail = 0;
    std::vector<int64_t> s(sources.begin(), sources.end()), t(targets.begin(), targets.end());
    check(recon_min_cost_1d(nullptr, static_cast<int32_t>(s.size()), s.data(), static_cast<int32_t>(t.size()),
                            t.data(), &cost, &detail),
          detail);
    return cost;
}

// Certified decomposition (exact1d.cpp:219-297, 409-428): candidate cuts at
// empty vertices, certified with exact optima computed on the device.
std::vector<Interval1D> decompose_1d(int n, const std::vector<int> &S, const std::vector<int> &T) {
    std::vector<int> s = S, t = T;
    std::sort(s.begin(), s.end());
    std::sort(t.begin(), t.end());
    {  // same checks and messages as assign_1d (validate_chain_instance)
        int64_t w;
        std::vector<int64_t> a(t.size() + 1), b(t.size() + 1);
        std::vector<int32_t> u(s.size() + 1);
        int32_t detail = 0;
        const recon_status st = recon_assign_1d(nullptr, n, s.data(), static_cast<int32_t>(s.size()), t.data(),
                                                static_cast<int32_t>(t.size()), &w, a.data(), b.data(), u.data(),
                                                &detail);
        if (st != RECON_OK) rethrow(st, detail);
    }
    if (t.empty()) return {};
    std::vector<char> is_s(static_cast<size_t>(n), 0), is_t(static_cast<size_t>(n), 0);
    for (int v : s) is_s[static_cast<size_t>(v)] = 1;
    for (int v : t) is_t[static_cast<size_t>(v)] = 1;
    struct Blk {
        std::vector<int> src, tgt;
    };
    std::vector<Blk> blocks;
    {
        const int E = static_cast<int>(s.size()) - static_cast<int>(t.size());
        int ps = 0, pt = 0, last = 0;
        Blk cur;
        for (int v = 0; v < n; ++v) {
            if (is_s[static_cast<size_t>(v)] || is_t[static_cast<size_t>(v)]) {
                if (is_s[static_cast<size_t>(v)]) cur.src.push_back(v), ++ps;
                if (is_t[static_cast<size_t>(v)]) cur.tgt.push_back(v), ++pt;
                continue;
            }
            const int D = ps - pt;
            if (D <= E && D >= last) {  // |cur.S| >= |cur.T| and suffix feasible
                last = D;
                if (!cur.src.empty() || !cur.tgt.empty()) blocks.push_back(cur);
                cur = Blk{};
            }
        }
        if (!cur.src.empty() || !cur.tgt.empty()) blocks.push_back(cur);
    }
    auto cost = [](const Blk &b) {
        return min_assignment_cost_1d(std::vector<long long>(b.src.begin(), b.src.end()),
                                      std::vector<long long>(b.tgt.begin(), b.tgt.end()));
    };
    if (blocks.size() > 1) {
        Blk whole{s, t};
        const long long global = cost(whole);
        std::vector<long long> w(blocks.size());
        long long sum = 0;
        for (size_t i = 0; i < blocks.size(); ++i) sum += (w[i] = cost(blocks[i]));
        if (sum != global) {
            size_t i = 0;
            while (i + 1 < blocks.size()) {
                Blk j = blocks[i];
                j.src.insert(j.src.end(), blocks[i + 1].src.begin(), blocks[i + 1].src.end());
                j.tgt.insert(j.tgt.end(), blocks[i + 1].tgt.begin(), blocks[i + 1].tgt.end());
                const long long wj = cost(j);
                if (wj < w[i] + w[i + 1]) {
                    blocks[i] = j;
                    w[i] = wj;
                    blocks.erase(blocks.begin() + static_cast<long>(i) + 1);
                    w.erase(w.begin() + static_cast<long>(i) + 1);
                    if (i > 0) --i;
                } else {
                    ++i;
                }
            }
            if (std::accumulate(w.begin(), w.end(), 0LL) != global) blocks = {whole};
        }
    }
    std::vector<Interval1D> out;
    for (const Blk &b : blocks) {
        if (b.tgt.empty()) continue;
        Interval1D iv;
        iv.sources = b.src;
        iv.targets = b.tgt;
        iv.lo = std::min(b.src.front(), b.tgt.front());
        iv.hi = std::max(b.src.back(), b.tgt.back());
        out.push_back(std::move(iv));
    }
    return out;
}

std::vector<Path> paths_from_matching(const Geometry &g, const Matching1D &m) {
    if (g.height != 1) throw InputError("1D paths require a chain geometry");
    std::vector<Path> paths;
    for (const auto &[sp, tp] : m.pairs) {
        const int s = static_cast<int>(sp), t = static_cast<int>(tp);
        if (s < 0 || s >= g.width || t < 0 || t >= g.width) throw InputError("matched position outside the chain");
        Path p;
        p.orientation = t > s ? Orientation::right : (t < s ? Orientation::left : Orientation::isolated);
        const int step = t > s ? 1 : -1;
        p.vertices.push_back(s);
        for (int v = s; v != t;) p.vertices.push_back(v += step);
        p.event_id = 0;
        p.src_column = s;
        p.dst_column = t;
        paths.push_back(std::move(p));
    }
    return paths;
}

std::vector<Path> resolve_nesting(std::vector<Path> paths) {
    // per orientation class: sources and targets re-paired in sorted order
    for (Orientation o : {Orientation::right, Orientation::left}) {
        const bool asc = o == Orientation::right;
        std::vector<size_t> ids;
        std::vector<int> srcs, tgts;
        for (size_t i = 0; i < paths.size(); ++i)
            if (paths[i].orientation == o) {
                ids.push_back(i);
                srcs.push_back(paths[i].source());
                tgts.push_back(paths[i].target());
            }
        std::sort(srcs.begin(), srcs.end());
        std::sort(tgts.begin(), tgts.end());
        if (!asc) {
            std::reverse(srcs.begin(), srcs.end());
            std::reverse(tgts.begin(), tgts.end());
        }
        std::stable_sort(ids.begin(), ids.end(), [&](size_t a, size_t b) {
            return asc ? paths[a].source() < paths[b].source() : paths[a].source() > paths[b].source();
        });
        for (size_t k = 0; k < ids.size(); ++k) {
            Path &p = paths[ids[k]];
            const int s = srcs[k], t = tgts[k], step = t > s ? 1 : -1;
            p.vertices.assign(1, s);
            for (int v = s; v != t;) p.vertices.push_back(v += step);
            p.dst_column = t;
        }
    }
    return paths;
}

std::vector<int> order_1d_intervals(const std::vector<std::pair<long long, long long>> &iv) {
    std::vector<int> rights, lefts, iso;
    for (size_t i = 0; i < iv.size(); ++i)
        (iv[i].second > iv[i].first ? rights : (iv[i].second < iv[i].first ? lefts : iso)).push_back(static_cast<int>(i));
    std::stable_sort(rights.begin(), rights.end(), [&](int a, int b) { return iv[static_cast<size_t>(a)].second > iv[static_cast<size_t>(b)].second; });
    std::stable_sort(lefts.begin(), lefts.end(), [&](int a, int b) { return iv[static_cast<size_t>(a)].second < iv[static_cast<size_t>(b)].second; });
    rights.insert(rights.end(), lefts.begin(), lefts.end());
    rights.insert(rights.end(), iso.begin(), iso.end());
    return rights;
}

Ordering1D order_moves_1d(const std::vector<Path> &paths) {
    std::vector<std::pair<long long, long long>> iv;
    for (const Path &p : paths) iv.emplace_back(p.source(), p.target());
    Ordering1D out;
    out.path_order = order_1d_intervals(iv);
    for (int id : out.path_order)
        for (const ElementaryMove &mv : moves_of(paths[static_cast<size_t>(id)])) out.schedule.push_back(mv);
    out.dag.node_count = static_cast<int>(paths.size());
    std::vector<int> rank(paths.size());
    for (size_t k = 0; k < out.path_order.size(); ++k) rank[static_cast<size_t>(out.path_order[k])] = static_cast<int>(k);
    // spans swept by (lo, id); earlier spans still reaching lo, by (hi, arrival)
    std::vector<int> ids(paths.size());
    std::iota(ids.begin(), ids.end(), 0);
    auto lo = [&](int i) { return std::min(iv[static_cast<size_t>(i)].first, iv[static_cast<size_t>(i)].second); };
    auto hi = [&](int i) { return std::max(iv[static_cast<size_t>(i)].first, iv[static_cast<size_t>(i)].second); };
    std::stable_sort(ids.begin(), ids.end(), [&](int a, int b) { return lo(a) < lo(b); });
    std::vector<int> active;  // kept ordered by (hi, arrival)
    for (int me : ids) {
        active.erase(active.begin(), std::find_if(active.begin(), active.end(), [&](int o) { return hi(o) >= lo(me); }));
        for (int other : active) {
            const int a = rank[static_cast<size_t>(other)] < rank[static_cast<size_t>(me)] ? other : me;
            out.dag.add_edge(a, a == other ? me : other);
        }
        auto at = std::find_if(active.begin(), active.end(), [&](int o) { return hi(o) > hi(me); });
        active.insert(at, me);
    }
    return out;
}

Solution solve_1d(int n, const std::vector<int> &S, const std::vector<int> &T) {
    const size_t nt = T.size();
    std::vector<int32_t> src(nt + 1), dst(nt + 1), order(nt + 1);
    int64_t dag_cap = 8 * static_cast<int64_t>(nt) + 64, dag_count = 0, total = 0;
    int32_t displaced = 0;
    for (;;) {
        std::vector<int32_t> da(static_cast<size_t>(dag_cap)), db(static_cast<size_t>(dag_cap));
        int32_t detail = 0;
        const recon_status st = recon_solve_1d(nullptr, n, S.data(), static_cast<int32_t>(S.size()), T.data(),
                                               static_cast<int32_t>(nt), src.data(), dst.data(), order.data(),
                                               da.data(), db.data(), dag_cap, &dag_count, &total, &displaced,
                                               &detail);
        if (st == RECON_ERR_CAPACITY && dag_count > dag_cap) {
            dag_cap = dag_count;
            continue;
        }
        check(st, detail);
        PathSystem ps;
        for (size_t i = 0; i < nt; ++i) {
            Path p;
            const int s = src[i], t = dst[i], step = t > s ? 1 : -1;
            p.orientation = t > s ? Orientation::right : (t < s ? Orientation::left : Orientation::isolated);
            p.vertices.assign(1, s);
            for (int v = s; v != t;) p.vertices.push_back(v += step);
            p.event_id = 0;
            p.src_column = s;
            p.dst_column = t;
            ps.paths.push_back(std::move(p));
        }
        MoveDag dag;
        dag.node_count = static_cast<int>(nt);
        for (int64_t e = 0; e < dag_count; ++e) dag.add_edge(da[static_cast<size_t>(e)], db[static_cast<size_t>(e)]);
        return make_solution(std::move(ps), std::move(dag), std::vector<int>(order.begin(), order.begin() + static_cast<long>(nt)));
    }
}

// ===========================================================================
// virtual_line.hpp
// ===========================================================================

BandSpec derive_centered_band(const Problem &problem) {
    const Geometry &g = problem.geometry;
    int y_lo, y_hi;
    if (problem.target_region) {
        y_lo = problem.target_region->row_lo(g);
        y_hi = problem.target_region->row_hi(g);
    } else {
        if (problem.targets.empty()) throw InputError("target band is empty");
        std::vector<std::vector<int>> rows(static_cast<size_t>(g.width));
        for (Vertex v : problem.targets.vertices()) rows[static_cast<size_t>(g.coords(v).x)].push_back(g.coords(v).y);
        const std::vector<int> &c0 = rows[0];
        if (c0.empty()) throw InputError("targets must form a centered full-width band");
        y_lo = c0.front();
        y_hi = c0.back();
        if (y_hi - y_lo + 1 != static_cast<int>(c0.size())) throw InputError("targets must form a centered full-width band");
        for (const auto &col : rows)
            if (col != c0) throw InputError("targets must form a centered full-width band");
        if (y_lo != (g.height - (y_hi - y_lo + 1)) / 2) throw InputError("targets must form a centered full-width band");
    }
    const int hp = y_hi - y_lo + 1;
    if (hp <= 0 || hp >= g.height) throw InputError("target band height must be in (0, H)");
    return BandSpec{g.row_from_top(y_hi), g.row_from_top(y_lo)};
}

SurplusVector compute_surpluses(const Problem &problem) {
    const BandSpec band = derive_centered_band(problem);
    SurplusVector s(static_cast<size_t>(problem.geometry.width), -band.h_prime());
    for (Vertex v : problem.sources.vertices()) ++s[static_cast<size_t>(problem.geometry.coords(v).x)];
    return s;
}

long long virtual_pos(const VirtualToken &token) { return vpos_of(token); }

VirtualToken virtual_token_at(const Geometry &g, BandSpec band, Vertex vertex, int receiver, bool mandatory) {
    const Vec2 p = g.coords(vertex);
    VirtualToken t;
    t.vertex = vertex;
    t.column = p.x;
    t.depth = g.row_from_top(p.y);
    t.dist = std::abs(p.x - receiver);
    t.top_side = t.depth < band.lo;
    t.mandatory = mandatory;
    return t;
}

VirtualToken virtual_token_at_depth(const Geometry &g, BandSpec band, int column, int depth, int receiver,
                                    bool mandatory) {
    return virtual_token_at(g, band, g.id({column, g.y_of_top_row(depth)}), receiver, mandatory);
}

std::vector<VirtualToken> own_column_tokens(const Geometry &g, BandSpec band, int column,
                                            const std::vector<int> &depths) {
    std::vector<VirtualToken> out;
    for (int d : depths) out.push_back(virtual_token_at_depth(g, band, column, d, column, band.contains(d)));
    return out;
}

VirtualEvent build_virtual_event(const Geometry &g, int receiver, BandSpec band, std::vector<VirtualToken> tokens) {
    std::stable_sort(tokens.begin(), tokens.end(), [](const VirtualToken &a, const VirtualToken &b) {
        const long long pa = vpos_of(a), pb = vpos_of(b);
        if (pa != pb) return pa < pb;
        if (a.dist != b.dist) return a.dist < b.dist;
        if (a.column != b.column) return a.column < b.column;
        return a.vertex < b.vertex;
    });
    VirtualEvent ev;
    ev.receiver = receiver;
    ev.band = band;
    ev.instance.offset = -(g.width - 1);
    ev.instance.length = g.height + 2 * (g.width - 1);
    for (int d = band.lo; d <= band.hi; ++d) ev.instance.targets.push_back(d);
    for (size_t i = 0; i < tokens.size();) {
        const long long pos = vpos_of(tokens[i]);
        Generalized1DSource src{pos, 0, 0};
        ev.origins.emplace_back();
        for (; i < tokens.size() && vpos_of(tokens[i]) == pos; ++i) {
            ++src.multiplicity;
            src.min_use += tokens[i].mandatory ? 1 : 0;
            ev.origins.back().push_back(tokens[i]);
        }
        ev.instance.sources.push_back(src);
    }
    return ev;
}

RealizedEvent realize_event(const Geometry &g, const VirtualEvent &event, const Matching1D &m, int event_id) {
    std::map<long long, size_t> group;
    for (size_t i = 0; i < event.instance.sources.size(); ++i) group[event.instance.sources[i].pos] = i;
    std::vector<std::vector<long long>> served(event.instance.sources.size());
    for (const auto &[pos, tgt] : m.pairs) served[group.at(pos)].push_back(tgt);
    RealizedEvent out;
    std::vector<std::pair<long long, long long>> iv;
    std::vector<Path> unordered;
    for (size_t i = 0; i < event.origins.size(); ++i) {
        std::sort(served[i].begin(), served[i].end());
        int optional = m.use_count[i] - event.instance.sources[i].min_use;
        std::vector<VirtualToken> drawn;
        for (const VirtualToken &t : event.origins[i]) {
            if (t.mandatory || optional > 0) {
                if (!t.mandatory) --optional;
                drawn.push_back(t);
            } else {
                out.parked.push_back(t);
            }
        }
        for (size_t k = 0; k < drawn.size(); ++k) {
            const long long tgt = served[i][k];
            out.placed.push_back(drawn[k]);
            if (vpos_of(drawn[k]) == tgt) continue;
            Path p;
            p.vertices = staircase(g, drawn[k].vertex, g.id({event.receiver, g.y_of_top_row(static_cast<int>(tgt))}));
            p.orientation = tgt > vpos_of(drawn[k]) ? Orientation::right : Orientation::left;
            p.src_column = drawn[k].column;
            p.dst_column = event.receiver;
            p.event_id = event_id;
            iv.emplace_back(vpos_of(drawn[k]), tgt);
            unordered.push_back(std::move(p));
        }
    }
    for (int idx : order_1d_intervals(iv)) out.paths.push_back(std::move(unordered[static_cast<size_t>(idx)]));
    return out;
}

MoveDag occupancy_dag(const std::vector<Path> &paths) {
    MoveDag dag;
    dag.node_count = static_cast<int>(paths.size());
    if (paths.empty()) return dag;
    Vertex vmax = 0;
    for (const Path &p : paths)
        for (Vertex v : p.vertices) vmax = std::max(vmax, v);
    std::vector<int64_t> off(paths.size() + 1, 0);
    std::vector<int32_t> verts;
    for (size_t i = 0; i < paths.size(); ++i) {
        verts.insert(verts.end(), paths[i].vertices.begin(), paths[i].vertices.end());
        off[i + 1] = static_cast<int64_t>(verts.size());
    }
    int64_t cap = 4 * static_cast<int64_t>(verts.size()) + 64, cnt = 0;
    for (;;) {
        std::vector<int32_t> a(static_cast<size_t>(cap)), b(static_cast<size_t>(cap));
        int32_t detail = 0;
        // vertex ids only index lookup planes: a 1 x (vmax+1) "grid" suffices
        const recon_status st = recon_occupancy_dag_paths(nullptr, vmax + 1, 1, static_cast<int32_t>(paths.size()),
                                                          off.data(), verts.data(), a.data(), b.data(), cap, &cnt,
                                                          &detail);
        if (st == RECON_ERR_CAPACITY && cnt > cap) {
            cap = cnt;
            continue;
        }
        check(st, detail);
        for (int64_t e = 0; e < cnt; ++e) dag.add_edge(a[static_cast<size_t>(e)], b[static_cast<size_t>(e)]);
        return dag;
    }
}

Solution assemble_event_solution(std::vector<Path> paths) {
    MoveDag dag = occupancy_dag(paths);
    std::vector<int> order(paths.size());
    std::iota(order.begin(), order.end(), 0);
    PathSystem ps;
    ps.paths = std::move(paths);
    return make_solution(std::move(ps), std::move(dag), order);
}

// ===========================================================================
// redrec.hpp
// ===========================================================================

RedRecState RedRecState::from_problem(const Problem &problem) {
    RedRecState st;
    st.geometry = problem.geometry;
    st.band = derive_centered_band(problem);
    const int W = st.geometry.width;
    st.column_depths.assign(static_cast<size_t>(W), {});
    st.marks_for.assign(static_cast<size_t>(W), {});
    for (Vertex v : problem.sources.vertices()) {
        const Vec2 p = st.geometry.coords(v);
        st.column_depths[static_cast<size_t>(p.x)].push_back(st.geometry.row_from_top(p.y));
    }
    st.surplus.assign(static_cast<size_t>(W), 0);
    for (int c = 0; c < W; ++c) {
        auto &d = st.column_depths[static_cast<size_t>(c)];
        std::sort(d.begin(), d.end());
        st.surplus[static_cast<size_t>(c)] = static_cast<int>(d.size()) - st.band.h_prime();
    }
    st.solved.assign(static_cast<size_t>(W), 0);
    return st;
}

std::pair<int, int> select_best_pair(const RedRecState &st) {
    const int W = st.geometry.width;
    auto donor_on = [&](int r, int step) {
        for (int c = r + step; c >= 0 && c < W; c += step) {
            const bool solved = st.solved[static_cast<size_t>(c)];
            const int s = st.surplus[static_cast<size_t>(c)];
            if (!solved && s > 0) return c;
            if (!(solved && s == 0)) return -1;
        }
        return -1;
    };
    bool any_receiver = false, found = false;
    std::array<int, 5> best{};
    for (int r = 0; r < W; ++r) {
        if (st.solved[static_cast<size_t>(r)] || st.surplus[static_cast<size_t>(r)] >= 0) continue;
        any_receiver = true;
        for (int step : {-1, +1}) {
            const int d = donor_on(r, step);
            if (d < 0) continue;
            const int deficit = -st.surplus[static_cast<size_t>(r)];
            const int ex = std::min(st.surplus[static_cast<size_t>(d)], deficit);
            const std::array<int, 5> key{-ex, std::abs(d - r), deficit - ex, r, d};
            if (!found || key < best) {
                best = key;
                found = true;
            }
        }
    }
    if (!any_receiver) throw std::logic_error("select_best_pair: no deficit column remains");
    if (!found) throw std::logic_error("select_best_pair: deficit column with no admissible donor");
    return {best[4], best[3]};
}

VirtualEvent build_redistribution_instance(int donor, int receiver, const RedRecState &st) {
    const Geometry &g = st.geometry;
    if (st.solved[static_cast<size_t>(receiver)]) {
        VirtualEvent e;
        e.receiver = receiver;
        e.band = st.band;
        e.instance.offset = -(g.width - 1);
        e.instance.length = g.height + 2 * (g.width - 1);
        return e;
    }
    std::vector<VirtualToken> tokens;
    for (int d : st.column_depths[static_cast<size_t>(receiver)])
        tokens.push_back(virtual_token_at_depth(g, st.band, receiver, d, receiver, true));
    for (const DelayedMark &mk : st.marks_for[static_cast<size_t>(receiver)])
        tokens.push_back(virtual_token_at(g, st.band, mk.vertex, receiver, true));
    if (donor >= 0)
        for (int d : st.column_depths[static_cast<size_t>(donor)])
            if (!st.band.contains(d)) tokens.push_back(virtual_token_at_depth(g, st.band, donor, d, receiver, false));
    return build_virtual_event(g, receiver, st.band, std::move(tokens));
}

Solution red_rec(const Problem &problem) { return red_rec(problem, nullptr); }

Solution red_rec(const Problem &problem, std::vector<RedRecEvent> *events) {
    std::vector<int32_t> ev;
    Solution sol = run_grid(
        problem,
        [](const uint64_t *occ, int W, int H, int k, recon_grid_solution *out, int32_t *detail) {
            return recon_redrec_solve(nullptr, occ, W, H, k, out, detail);
        },
        ev, 4);
    if (events) {
        events->clear();
        for (size_t i = 0; i + 3 < ev.size(); i += 4) events->push_back(RedRecEvent{ev[i], ev[i + 1], ev[i + 2], ev[i + 3]});
    }
    return sol;
}

// ===========================================================================
// bird.hpp
// ===========================================================================

BirdState BirdState::from_problem(const Problem &problem) {
    const RedRecState r = RedRecState::from_problem(problem);
    BirdState st;
    st.geometry = r.geometry;
    st.band = r.band;
    st.column_depths = r.column_depths;
    st.surplus = r.surplus;
    st.solved = r.solved;
    return st;
}

VirtualEvent build_generalized_instance(const BirdState &st, int column) {
    const Geometry &g = st.geometry;
    std::vector<VirtualToken> tokens = own_column_tokens(g, st.band, column, st.column_depths[static_cast<size_t>(column)]);
    for (int c = 0; c < g.width; ++c) {
        if (c == column) continue;
        for (int d : st.column_depths[static_cast<size_t>(c)])
            if (!st.band.contains(d)) tokens.push_back(virtual_token_at_depth(g, st.band, c, d, column, false));
    }
    return build_virtual_event(g, column, st.band, std::move(tokens));
}

Solution bird(const Problem &problem) { return bird(problem, nullptr); }

Solution bird(const Problem &problem, std::vector<int> *solved_order) {
    std::vector<int32_t> ev;
    Solution sol = run_grid(
        problem,
        [](const uint64_t *occ, int W, int H, int k, recon_grid_solution *out, int32_t *detail) {
            return recon_bird_solve(nullptr, occ, W, H, k, out, detail);
        },
        ev, 1);
    if (solved_order) solved_order->assign(ev.begin(), ev.end());
    return sol;
}

// ===========================================================================
// batching.hpp
// ===========================================================================

BatchDir move_dir(const Geometry &g, ElementaryMove m) {
    const Vec2 a = g.coords(m.from), b = g.coords(m.to);
    if (b.y > a.y) return BatchDir::up;
    if (b.y < a.y) return BatchDir::down;
    return b.x < a.x ? BatchDir::left : BatchDir::right;
}

bool ConstraintSet::compatible(const Geometry &g, ElementaryMove a, ElementaryMove b) const {
    if (preset == ConstraintPreset::none) return true;
    const BatchDir da = move_dir(g, a), db = move_dir(g, b);
    if (da != db) return false;
    const Vec2 fa = g.coords(a.from), fb = g.coords(b.from);
    return (da == BatchDir::up || da == BatchDir::down) ? fa.x == fb.x : fa.y == fb.y;
}

ConstraintSet deployed_constraint() { return ConstraintSet{ConstraintPreset::column_direction}; }

BatchSchedule batch_moves(const Problem &problem, const Solution &solution, const BatchOptions &options) {
    const Geometry &g = problem.geometry;
    const auto &paths = solution.path_system.paths;
    const std::vector<uint64_t> occ = pack_grid(g, problem.sources);
    std::vector<int64_t> off(paths.size() + 1, 0);
    std::vector<int32_t> verts;
    for (size_t i = 0; i < paths.size(); ++i) {
        verts.insert(verts.end(), paths[i].vertices.begin(), paths[i].vertices.end());
        off[i + 1] = static_cast<int64_t>(verts.size());
    }
    std::vector<int32_t> es, ed;
    for (const auto &[a, b] : solution.dag.edges) {
        es.push_back(a);
        ed.push_back(b);
    }
    if (solution.dag.node_count != static_cast<int>(paths.size())) {
        // MoveDag::topo_order validates endpoints against node_count (path_system.cpp:11-12)
        for (size_t e = 0; e < es.size(); ++e)
            if (es[e] >= solution.dag.node_count || ed[e] >= solution.dag.node_count)
                throw InputError("batching requires an acyclic dependency dag");
    }
    const int64_t moves = off.back() - static_cast<int64_t>(paths.size());
    std::vector<int32_t> mb(static_cast<size_t>(std::max<int64_t>(moves, 1)));
    int64_t nb = 0;
    int32_t detail = 0;
    const int preset = options.constraints.preset == ConstraintPreset::column_direction ? RECON_PRESET_COLUMN_DIRECTION
                                                                                         : RECON_PRESET_NONE;
    check(recon_batch_moves(nullptr, g.width, g.height, occ.data(), static_cast<int32_t>(paths.size()), off.data(),
                            verts.data(), static_cast<int64_t>(es.size()), es.data(), ed.data(), preset,
                            options.edge_level ? 1 : 0, mb.data(), &nb, &detail),
          detail);
    BatchSchedule out;
    out.batches.resize(static_cast<size_t>(nb));
    for (size_t p = 0; p < paths.size(); ++p)  // ascending path id within each batch
        for (int k = 0; k < paths[p].length(); ++k) {
            const int b = mb[static_cast<size_t>(off[p] - static_cast<int64_t>(p) + k)];
            out.batches[static_cast<size_t>(b)].moves.push_back({paths[p].vertices[static_cast<size_t>(k)],
                                                                 paths[p].vertices[static_cast<size_t>(k) + 1]});
        }
    if (options.constraints.preset != ConstraintPreset::none)
        for (Batch &b : out.batches) {
            b.dir = move_dir(g, b.moves.front());
            b.axis = (b.dir == BatchDir::up || b.dir == BatchDir::down) ? BatchAxis::col : BatchAxis::row;
        }
    return out;
}

// Batch-schedule verifier (host; not on the solve path).
ValidationReport validate_batches(const Problem &problem, const Solution &solution, const BatchSchedule &schedule,
                                  const BatchOptions &options) {
    ValidationReport rep;
    const Geometry &g = problem.geometry;
    std::map<std::pair<Vertex, Vertex>, long long> balance;
    for (const Path &p : solution.path_system.paths)
        for (const ElementaryMove &m : moves_of(p)) ++balance[{m.from, m.to}];
    for (const Batch &b : schedule.batches)
        for (const ElementaryMove &m : b.moves) --balance[{m.from, m.to}];
    for (const auto &kv : balance)
        if (kv.second != 0) {
            rep.fail("batched moves do not conserve the path-system edge multiset");
            break;
        }
    if (static_cast<long long>(schedule.batches.size()) > solution.path_system.weight())
        rep.fail("more batches than elementary moves");
    Configuration occ = problem.sources;
    for (size_t bi = 0; bi < schedule.batches.size(); ++bi) {
        const Batch &b = schedule.batches[bi];
        const std::string tag = "batch " + std::to_string(bi);
        if (b.moves.empty()) {
            rep.fail(tag + " is empty");
            continue;
        }
        std::vector<char> used(static_cast<size_t>(g.size()), 0);
        for (const ElementaryMove &m : b.moves) {
            if (!g.in_bounds(m.from) || !g.in_bounds(m.to) || !g.adjacent(m.from, m.to)) {
                rep.fail(tag + " contains a non-elementary move");
                return rep;
            }
            if (used[static_cast<size_t>(m.from)] || used[static_cast<size_t>(m.to)]) {
                rep.fail(tag + " is not vertex-disjoint");
                return rep;
            }
            used[static_cast<size_t>(m.from)] = used[static_cast<size_t>(m.to)] = 1;
        }
        bool ok = true;
        for (size_t i = 0; i < b.moves.size() && ok; ++i)
            for (size_t j = i + 1; j < b.moves.size() && ok; ++j)
                ok = options.constraints.compatible(g, b.moves[i], b.moves[j]);
        if (!ok) rep.fail(tag + " violates the constraint set");
        for (const ElementaryMove &m : b.moves) {
            if (!occ.contains(m.from)) {
                rep.fail(tag + " moves a token from an empty vertex");
                return rep;
            }
            if (occ.contains(m.to)) {
                rep.fail(tag + " moves into a vertex occupied before the batch");
                return rep;
            }
        }
        for (const ElementaryMove &m : b.moves) occ.remove(m.from);
        for (const ElementaryMove &m : b.moves) occ.add(m.to);
    }
    if (!occ.contains_all(problem.targets)) rep.fail("batched execution does not cover all targets");
    if (!rep.pass) return rep;
    std::vector<ElementaryMove> flat;
    std::vector<size_t> batch_of;
    for (size_t bi = 0; bi < schedule.batches.size(); ++bi)
        for (const ElementaryMove &m : schedule.batches[bi].moves) {
            flat.push_back(m);
            batch_of.push_back(bi);
        }
    auto match = match_schedule(solution.path_system, flat, rep);
    if (!match) return rep;
    for (const auto &[i, j] : solution.dag.edges) {
        const int fi = match->first_move[static_cast<size_t>(i)], fj = match->first_move[static_cast<size_t>(j)];
        if (fi >= 0 && fj >= 0 && batch_of[static_cast<size_t>(fj)] < batch_of[static_cast<size_t>(fi)]) {
            rep.fail("batch order violates dag edge " + std::to_string(i) + "->" + std::to_string(j));
            break;
        }
    }
    return rep;
}

}  // namespace recon
