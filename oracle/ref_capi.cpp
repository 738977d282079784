// oracle/ref_capi.cpp — TEST INFRASTRUCTURE, not product code.
//
// Exposes the UNMODIFIED reference implementation (/root/reference/proj,
// compiled from its own sources by oracle/Makefile into oracle/_ref/) behind
// the same C-ABI as the B200 library (include/recon_b200.h), so the parity
// tests and bench.py's CPU-baseline leg can drive the reference and the GPU
// path with identical buffers.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load this library.
//
// Every function here is a thin marshalling layer: decode the C buffers into
// the reference's own types, call the reference's public API, encode the
// result.  "Device" pointers of the *_batch entry points are host pointers
// for this CPU library.

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "digest_cpu.h"

#include "recon/batching.hpp"
#include "recon/bird.hpp"
#include "recon/exact1d.hpp"
#include "recon/redrec.hpp"
#include "recon/rng.hpp"
#include "recon/virtual_line.hpp"
#include "recon_b200.h"

using namespace recon;

struct recon_ctx {
    int device = 0;
};

namespace {

struct Failure {
    recon_status status;
    int32_t detail;
};

int32_t detail_of_message(const std::string &m) {
    static const std::pair<const char *, int32_t> table[] = {
        {"fewer sources than targets (|S| < |T|)", RECON_D_FEWER_SOURCES},
        {"targets must form a centered full-width band", RECON_D_BAND_NOT_CENTERED},
        {"target band height must be in (0, H)", RECON_D_BAND_HEIGHT},
        {"target region height must be in (0, H)", RECON_D_BAND_HEIGHT},
        {"target band is empty", RECON_D_BAND_EMPTY},
        {"select_best_pair: no deficit column remains", RECON_D_NO_DEFICIT},
        {"select_best_pair: deficit column with no admissible donor", RECON_D_NO_DONOR},
        {"batching made no progress (blocked dependency structure)", RECON_D_BATCH_NO_PROGRESS},
        {"batching requires an acyclic dependency dag", RECON_D_BATCH_CYCLIC},
        {"chain length must be positive", RECON_D_CHAIN_LENGTH},
        {"source vertex out of bounds", RECON_D_SOURCE_OOB},
        {"source vertices must be strictly increasing", RECON_D_SOURCE_ORDER},
        {"target vertex out of bounds", RECON_D_TARGET_OOB},
        {"target vertices must be strictly increasing", RECON_D_TARGET_ORDER},
        {"source multiplicity must be at least 1", RECON_D_GEN_MULTIPLICITY},
        {"source min_use outside [0, multiplicity]", RECON_D_GEN_MIN_USE},
        {"source positions must be strictly increasing", RECON_D_GEN_SOURCE_ORDER},
        {"target positions must be strictly increasing", RECON_D_GEN_TARGET_ORDER},
        {"insufficient tokens for targets", RECON_D_GEN_SUPPLY},
        {"mandatory draws exceed target count", RECON_D_GEN_MANDATORY},
        {"no assignment satisfies the usage bounds", RECON_D_GEN_NO_ASSIGNMENT},
        {"dag edge endpoint out of range", RECON_D_DAG_EDGE_RANGE},
        {"grid dimensions must be positive", RECON_D_GRID_DIMENSIONS},
        {"fewer sources than targets", RECON_D_INFEASIBLE_SUPPLY},
    };
    for (const auto &[msg, d] : table)
        if (m == msg) return d;
    return RECON_D_NONE;
}

template <typename F>
recon_status guarded(int32_t *detail, F &&f) {
    if (detail) *detail = RECON_D_NONE;
    try {
        f();
        return RECON_OK;
    } catch (const Failure &e) {
        if (detail) *detail = e.detail;
        return e.status;
    } catch (const InputError &e) {
        if (detail) *detail = detail_of_message(e.what());
        return RECON_ERR_INPUT;
    } catch (const InfeasibleError &e) {
        if (detail) *detail = detail_of_message(e.what());
        return RECON_ERR_INFEASIBLE;
    } catch (const CollisionError &e) {
        if (detail) *detail = detail_of_message(e.what());
        return RECON_ERR_COLLISION;
    } catch (const std::logic_error &e) {
        if (detail) *detail = detail_of_message(e.what());
        return RECON_ERR_LOGIC;
    }
}

int words_per_column(int h) { return (h + 63) / 64; }

std::vector<Vertex> decode_grid(const uint64_t *occ, int w, int h) {
    const int wpc = words_per_column(h);
    std::vector<Vertex> S;
    for (int x = 0; x < w; ++x)
        for (int y = 0; y < h; ++y)
            if ((occ[static_cast<size_t>(x) * wpc + y / 64] >> (y % 64)) & 1ULL)
                S.push_back(static_cast<Vertex>(x * h + y));
    return S;
}

std::vector<int> decode_chain(const uint64_t *occ, int n) {
    std::vector<int> S;
    for (int v = 0; v < n; ++v)
        if ((occ[v / 64] >> (v % 64)) & 1ULL) S.push_back(v);
    return S;
}

Path one_bend_path(const Geometry &g, Vertex s, Vertex t) {
    Path p;
    for (const Vec2 &v : shortest_path(g.coords(s), g.coords(t), StepPolicy::horizontal_first))
        p.vertices.push_back(g.id(v));
    return p;
}

int ref_threads() {
    const char *env = std::getenv("RECON_REF_THREADS");
    int n = env ? std::atoi(env) : 0;
    if (n <= 0) n = static_cast<int>(std::thread::hardware_concurrency());
    return std::max(1, n);
}

template <typename F>
void parallel_for(int count, F &&f) {
    const int nt = std::min(ref_threads(), std::max(1, count));
    if (nt <= 1) {
        for (int i = 0; i < count; ++i) f(i);
        return;
    }
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&] {
            for (int i = next++; i < count; i = next++) f(i);
        });
    for (auto &th : pool) th.join();
}

void write_grid_solution(const Solution &sol, recon_grid_solution *out) {
    const auto &paths = sol.path_system.paths;
    out->path_count = static_cast<int64_t>(paths.size());
    out->displaced_tokens = sol.stats.displaced_tokens;
    out->total_displacement = sol.stats.total_displacement;
    if (static_cast<int64_t>(paths.size()) > out->path_capacity)
        throw Failure{RECON_ERR_CAPACITY, RECON_D_NONE};
    for (size_t i = 0; i < paths.size(); ++i) {
        out->path_src[i] = paths[i].source();
        out->path_dst[i] = paths[i].target();
        if (out->path_event) out->path_event[i] = paths[i].event_id;
    }
    if (out->dag_src) {
        out->dag_count = static_cast<int64_t>(sol.dag.edges.size());
        if (out->dag_count > out->dag_capacity) throw Failure{RECON_ERR_CAPACITY, RECON_D_NONE};
        for (size_t i = 0; i < sol.dag.edges.size(); ++i) {
            out->dag_src[i] = sol.dag.edges[i].first;
            out->dag_dst[i] = sol.dag.edges[i].second;
        }
    }
}

Problem grid_problem(const uint64_t *occ, int w, int h, int h_prime) {
    return Problem::make_centered(Geometry::grid(w, h), decode_grid(occ, w, h), h_prime);
}

recon_status grid_batch(const recon_grid_batch *b, bool pooled) {
    if (!b || !b->occ) return RECON_ERR_ARGUMENT;
    const int wpc = words_per_column(b->height);
    const int64_t stride = static_cast<int64_t>(b->width) * b->h_prime;
    parallel_for(b->count, [&](int i) {
        recon_grid_solution out{};
        out.path_src = b->path_src + i * stride;
        out.path_dst = b->path_dst + i * stride;
        out.path_event = b->path_event ? b->path_event + i * stride : nullptr;
        out.path_capacity = stride;
        std::vector<int32_t> ev(static_cast<size_t>(b->width) * 4);
        int32_t detail = 0;
        const uint64_t *occ = b->occ + static_cast<size_t>(i) * b->width * wpc;
        recon_status st = guarded(&detail, [&] {
            const Problem p = grid_problem(occ, b->width, b->height, b->h_prime);
            if (pooled) {
                std::vector<int> order;
                write_grid_solution(recon::bird(p, &order), &out);
                if (b->events)
                    for (size_t k = 0; k < order.size(); ++k)
                        b->events[static_cast<size_t>(i) * b->width + k] = order[k];
            } else {
                std::vector<RedRecEvent> events;
                write_grid_solution(recon::red_rec(p, &events), &out);
                if (b->events)
                    for (size_t k = 0; k < events.size(); ++k) {
                        int32_t *e = b->events + (static_cast<size_t>(i) * b->width + k) * 4;
                        e[0] = events[k].event_id;
                        e[1] = events[k].column;
                        e[2] = events[k].donor;
                        e[3] = events[k].mark_destination;
                    }
            }
        });
        b->path_count[i] = st == RECON_OK ? static_cast<int32_t>(out.path_count) : 0;
        b->total_displacement[i] = st == RECON_OK ? out.total_displacement : 0;
        b->status[i] = st;
        if (b->detail) b->detail[i] = detail;
    });
    return RECON_OK;
}

BatchSchedule run_batching(const Problem &p, const Solution &sol, int32_t preset,
                           int32_t edge_level) {
    BatchOptions opt;
    opt.constraints.preset =
        preset == RECON_PRESET_COLUMN_DIRECTION ? ConstraintPreset::column_direction
                                                : ConstraintPreset::none;
    opt.edge_level = edge_level != 0;
    return batch_moves(p, sol, opt);
}

// Attributes each batched move to its path (moves of one batch are vertex
// disjoint, and pending path fronts sit on distinct vertices) and writes the
// batch index at the path-major move slot.
void encode_batches(const Solution &sol, const BatchSchedule &bs, int32_t *move_batch,
                    const std::vector<int64_t> &move_base) {
    const auto &paths = sol.path_system.paths;
    std::vector<size_t> next(paths.size(), 0);
    std::map<Vertex, std::vector<int>> pending;
    for (size_t i = 0; i < paths.size(); ++i)
        if (paths[i].length() > 0) pending[paths[i].source()].push_back(static_cast<int>(i));
    for (size_t b = 0; b < bs.batches.size(); ++b) {
        std::vector<std::pair<int, Vertex>> advanced;
        for (const ElementaryMove &m : bs.batches[b].moves) {
            auto it = pending.find(m.from);
            int pid = -1;
            if (it != pending.end())
                for (int cand : it->second)
                    if (paths[static_cast<size_t>(cand)].vertices[next[static_cast<size_t>(cand)] + 1] == m.to) {
                        pid = cand;
                        break;
                    }
            if (pid < 0) throw std::runtime_error("ref_capi: unattributable batched move");
            auto &ids = it->second;
            ids.erase(std::find(ids.begin(), ids.end(), pid));
            if (ids.empty()) pending.erase(it);
            move_batch[move_base[static_cast<size_t>(pid)] + static_cast<int64_t>(next[static_cast<size_t>(pid)])] =
                static_cast<int32_t>(b);
            const size_t k = ++next[static_cast<size_t>(pid)];
            if (k < static_cast<size_t>(paths[static_cast<size_t>(pid)].length()))
                advanced.emplace_back(pid, paths[static_cast<size_t>(pid)].vertices[k]);
        }
        for (auto [pid, v] : advanced) pending[v].push_back(pid);
    }
}

}  // namespace

extern "C" {

const char *recon_detail_message(int32_t detail) {
    switch (detail) {
        case RECON_D_FEWER_SOURCES: return "fewer sources than targets (|S| < |T|)";
        case RECON_D_BAND_NOT_CENTERED: return "targets must form a centered full-width band";
        case RECON_D_BAND_HEIGHT: return "target band height must be in (0, H)";
        case RECON_D_BAND_EMPTY: return "target band is empty";
        case RECON_D_NO_DEFICIT: return "select_best_pair: no deficit column remains";
        case RECON_D_NO_DONOR: return "select_best_pair: deficit column with no admissible donor";
        case RECON_D_BATCH_NO_PROGRESS: return "batching made no progress (blocked dependency structure)";
        case RECON_D_BATCH_CYCLIC: return "batching requires an acyclic dependency dag";
        default: return "";
    }
}
const char *recon_last_cuda_error(void) { return ""; }
int32_t recon_abi_version(void) { return RECON_ABI_VERSION; }

recon_status recon_ctx_create(int32_t device, recon_ctx **out) {
    *out = new recon_ctx{device};
    return RECON_OK;
}
void recon_ctx_destroy(recon_ctx *ctx) { delete ctx; }
void *recon_ctx_stream(recon_ctx *) { return nullptr; }
int64_t recon_ctx_launch_count(recon_ctx *) { return 0; }
recon_status recon_ctx_set_kernel_timing(recon_ctx *, int32_t) { return RECON_OK; }
recon_status recon_ctx_kernel_times(recon_ctx *, float *ms, int32_t n) {
    for (int32_t i = 0; i < n; ++i) ms[i] = 0.0f;
    return RECON_OK;
}

recon_status recon_redrec_solve(recon_ctx *, const uint64_t *occ, int32_t width, int32_t height,
                                int32_t h_prime, recon_grid_solution *out, int32_t *detail) {
    return guarded(detail, [&] {
        const Problem p = grid_problem(occ, width, height, h_prime);
        std::vector<RedRecEvent> events;
        const Solution sol = red_rec(p, &events);
        out->event_count = static_cast<int32_t>(events.size());
        if (out->events) {
            if (static_cast<int32_t>(events.size()) * 4 > out->event_capacity)
                throw Failure{RECON_ERR_CAPACITY, RECON_D_NONE};
            for (size_t k = 0; k < events.size(); ++k) {
                out->events[4 * k] = events[k].event_id;
                out->events[4 * k + 1] = events[k].column;
                out->events[4 * k + 2] = events[k].donor;
                out->events[4 * k + 3] = events[k].mark_destination;
            }
        }
        write_grid_solution(sol, out);
    });
}

recon_status recon_bird_solve(recon_ctx *, const uint64_t *occ, int32_t width, int32_t height,
                              int32_t h_prime, recon_grid_solution *out, int32_t *detail) {
    return guarded(detail, [&] {
        const Problem p = grid_problem(occ, width, height, h_prime);
        std::vector<int> order;
        const Solution sol = bird(p, &order);
        out->event_count = static_cast<int32_t>(order.size());
        if (out->events) {
            if (static_cast<int32_t>(order.size()) > out->event_capacity)
                throw Failure{RECON_ERR_CAPACITY, RECON_D_NONE};
            for (size_t k = 0; k < order.size(); ++k) out->events[k] = order[k];
        }
        write_grid_solution(sol, out);
    });
}

recon_status recon_occupancy_dag(recon_ctx *, int32_t width, int32_t height,
                                 const int32_t *path_src, const int32_t *path_dst,
                                 int64_t path_count, int32_t *dag_src, int32_t *dag_dst,
                                 int64_t dag_capacity, int64_t *dag_count, int32_t *detail) {
    return guarded(detail, [&] {
        const Geometry g = Geometry::grid(width, height);
        std::vector<Path> paths;
        for (int64_t i = 0; i < path_count; ++i) paths.push_back(one_bend_path(g, path_src[i], path_dst[i]));
        const MoveDag dag = occupancy_dag(paths);
        *dag_count = static_cast<int64_t>(dag.edges.size());
        if (*dag_count > dag_capacity) throw Failure{RECON_ERR_CAPACITY, RECON_D_NONE};
        for (size_t i = 0; i < dag.edges.size(); ++i) {
            dag_src[i] = dag.edges[i].first;
            dag_dst[i] = dag.edges[i].second;
        }
    });
}

recon_status recon_redrec_solve_batch(recon_ctx *, const recon_grid_batch *b) { return grid_batch(b, false); }
recon_status recon_bird_solve_batch(recon_ctx *, const recon_grid_batch *b) { return grid_batch(b, true); }
recon_status recon_redrec_solve_batch_host(recon_ctx *, const recon_grid_batch *b) { return grid_batch(b, false); }
recon_status recon_bird_solve_batch_host(recon_ctx *, const recon_grid_batch *b) { return grid_batch(b, true); }

static recon_status grid_batch_packed(const recon_grid_batch *b, bool pooled, uint32_t *packed) {
    if (!packed || !b || static_cast<int64_t>(b->width) * b->height > 65536) return RECON_ERR_ARGUMENT;
    const size_t n = static_cast<size_t>(std::max(b->count, 0)) * b->width * b->h_prime;
    std::vector<int32_t> src(n), dst(n);
    recon_grid_batch t = *b;
    t.path_src = src.data();
    t.path_dst = dst.data();
    const recon_status st = grid_batch(&t, pooled);
    for (size_t i = 0; i < n; ++i) packed[i] = static_cast<uint32_t>(src[i]) | static_cast<uint32_t>(dst[i]) << 16;
    return st;
}
recon_status recon_redrec_solve_batch_host_packed(recon_ctx *, const recon_grid_batch *b, uint32_t *packed) {
    return grid_batch_packed(b, false, packed);
}
recon_status recon_bird_solve_batch_host_packed(recon_ctx *, const recon_grid_batch *b, uint32_t *packed) {
    return grid_batch_packed(b, true, packed);
}

recon_status recon_assign_1d(recon_ctx *, int32_t n, const int32_t *S, int32_t ns, const int32_t *T,
                             int32_t nt, int64_t *weight, int64_t *pair_src, int64_t *pair_dst,
                             int32_t *use_count, int32_t *detail) {
    return guarded(detail, [&] {
        const Matching1D m = assign_1d(n, std::vector<int>(S, S + ns), std::vector<int>(T, T + nt));
        *weight = m.weight;
        for (size_t i = 0; i < m.pairs.size(); ++i) {
            pair_src[i] = m.pairs[i].first;
            pair_dst[i] = m.pairs[i].second;
        }
        for (size_t i = 0; i < m.use_count.size(); ++i) use_count[i] = m.use_count[i];
    });
}

recon_status recon_assign_1d_generalized(recon_ctx *, int32_t nsrc, const int64_t *pos,
                                         const int32_t *multiplicity, const int32_t *min_use,
                                         int32_t nt, const int64_t *targets, int64_t *weight,
                                         int64_t *pair_src, int64_t *pair_dst,
                                         int32_t *use_count, int32_t *detail) {
    return guarded(detail, [&] {
        Generalized1DInstance inst;
        for (int32_t i = 0; i < nsrc; ++i) inst.sources.push_back({pos[i], multiplicity[i], min_use[i]});
        inst.targets.assign(targets, targets + nt);
        const Matching1D m = assign_1d_generalized(inst);
        *weight = m.weight;
        for (size_t i = 0; i < m.pairs.size(); ++i) {
            pair_src[i] = m.pairs[i].first;
            pair_dst[i] = m.pairs[i].second;
        }
        for (size_t i = 0; i < m.use_count.size(); ++i) use_count[i] = m.use_count[i];
    });
}

recon_status recon_solve_1d(recon_ctx *, int32_t n, const int32_t *S, int32_t ns, const int32_t *T,
                            int32_t nt, int32_t *path_src, int32_t *path_dst, int32_t *path_order,
                            int32_t *dag_src, int32_t *dag_dst, int64_t dag_capacity,
                            int64_t *dag_count, int64_t *total_displacement, int32_t *displaced,
                            int32_t *detail) {
    return guarded(detail, [&] {
        const Solution sol = solve_1d(n, std::vector<int>(S, S + ns), std::vector<int>(T, T + nt));
        const auto &paths = sol.path_system.paths;
        for (size_t i = 0; i < paths.size(); ++i) {
            path_src[i] = paths[i].source();
            path_dst[i] = paths[i].target();
        }
        // the execution order solve_1d used (exact1d.cpp:517-528 via the
        // reference's own public order_moves_1d)
        if (path_order) {
            const Ordering1D ord = order_moves_1d(paths);
            for (size_t k = 0; k < ord.path_order.size(); ++k) path_order[k] = ord.path_order[k];
        }
        if (dag_src) {
            *dag_count = static_cast<int64_t>(sol.dag.edges.size());
            if (*dag_count > dag_capacity) throw Failure{RECON_ERR_CAPACITY, RECON_D_NONE};
            for (size_t i = 0; i < sol.dag.edges.size(); ++i) {
                dag_src[i] = sol.dag.edges[i].first;
                dag_dst[i] = sol.dag.edges[i].second;
            }
        } else if (dag_count) {
            *dag_count = static_cast<int64_t>(sol.dag.edges.size());
        }
        *total_displacement = sol.stats.total_displacement;
        *displaced = sol.stats.displaced_tokens;
    });
}

static recon_status chain_batch(const recon_chain_batch *b) {
    if (!b || !b->occ) return RECON_ERR_ARGUMENT;
    const int wpn = (b->n + 63) / 64;
    const int nt = b->t_hi - b->t_lo + 1;
    std::vector<int> T(static_cast<size_t>(nt));
    for (int i = 0; i < nt; ++i) T[static_cast<size_t>(i)] = b->t_lo + i;
    parallel_for(b->count, [&](int i) {
        int32_t detail = 0;
        recon_status st = guarded(&detail, [&] {
            const std::vector<int> S = decode_chain(b->occ + static_cast<size_t>(i) * wpn, b->n);
            const Solution sol = solve_1d(b->n, S, T);
            const auto &paths = sol.path_system.paths;
            for (size_t k = 0; k < paths.size(); ++k) {
                b->path_src[static_cast<size_t>(i) * nt + k] = paths[k].source();
                b->path_dst[static_cast<size_t>(i) * nt + k] = paths[k].target();
            }
            b->total_displacement[i] = sol.stats.total_displacement;
            b->displaced[i] = sol.stats.displaced_tokens;
        });
        b->status[i] = st;
        if (b->detail) b->detail[i] = detail;
    });
    return RECON_OK;
}

recon_status recon_solve_1d_batch(recon_ctx *, const recon_chain_batch *b) { return chain_batch(b); }
recon_status recon_solve_1d_batch_host(recon_ctx *, const recon_chain_batch *b) { return chain_batch(b); }

recon_status recon_batch_moves(recon_ctx *, int32_t width, int32_t height, const uint64_t *occ,
                               int32_t path_count, const int64_t *path_offsets,
                               const int32_t *path_vertices, int64_t edge_count,
                               const int32_t *edge_src, const int32_t *edge_dst, int32_t preset,
                               int32_t edge_level, int32_t *move_batch, int64_t *batch_count,
                               int32_t *detail) {
    return guarded(detail, [&] {
        const Geometry g = Geometry::grid(width, height);
        Problem p;
        p.geometry = g;
        p.sources = Configuration::from_vertices(g.size(), decode_grid(occ, width, height));
        p.targets = Configuration(g.size());
        Solution sol;
        std::vector<int64_t> base(static_cast<size_t>(path_count));
        for (int32_t i = 0; i < path_count; ++i) {
            Path path;
            path.vertices.assign(path_vertices + path_offsets[i], path_vertices + path_offsets[i + 1]);
            sol.path_system.paths.push_back(std::move(path));
            base[static_cast<size_t>(i)] = path_offsets[i] - i;
        }
        sol.dag.node_count = path_count;
        for (int64_t e = 0; e < edge_count; ++e) sol.dag.add_edge(edge_src[e], edge_dst[e]);
        const BatchSchedule bs = run_batching(p, sol, preset, edge_level);
        *batch_count = static_cast<int64_t>(bs.batches.size());
        encode_batches(sol, bs, move_batch, base);
    });
}

recon_status recon_pipeline_batch_run(recon_ctx *, const recon_pipeline_batch *pb) {
    const recon_grid_batch *b = &pb->grid;
    if (!b || !b->occ) return RECON_ERR_ARGUMENT;
    const int wpc = words_per_column(b->height);
    const int64_t stride = static_cast<int64_t>(b->width) * b->h_prime;
    parallel_for(b->count, [&](int i) {
        int32_t detail = 0;
        int64_t pc = 0, td = 0, nb = 0;
        recon_status st = guarded(&detail, [&] {
            const Problem p = grid_problem(b->occ + static_cast<size_t>(i) * b->width * wpc,
                                           b->width, b->height, b->h_prime);
            const Solution sol = pb->solver == 1 ? recon::bird(p) : recon::red_rec(p);
            const auto &paths = sol.path_system.paths;
            pc = static_cast<int64_t>(paths.size());
            td = sol.stats.total_displacement;
            std::vector<int64_t> base(paths.size());
            int64_t acc = 0;
            for (size_t k = 0; k < paths.size(); ++k) {
                b->path_src[i * stride + static_cast<int64_t>(k)] = paths[k].source();
                b->path_dst[i * stride + static_cast<int64_t>(k)] = paths[k].target();
                if (b->path_event) b->path_event[i * stride + static_cast<int64_t>(k)] = paths[k].event_id;
                base[k] = acc;
                acc += paths[k].length();
            }
            if (acc > pb->move_stride) throw Failure{RECON_ERR_CAPACITY, RECON_D_NONE};
            const BatchSchedule bs = run_batching(p, sol, pb->preset, 0);
            nb = static_cast<int64_t>(bs.batches.size());
            encode_batches(sol, bs, pb->move_batch + i * pb->move_stride, base);
        });
        b->path_count[i] = static_cast<int32_t>(pc);
        b->total_displacement[i] = td;
        b->status[i] = st;
        if (b->detail) b->detail[i] = detail;
        pb->batch_count[i] = static_cast<int32_t>(nb);
    });
    return RECON_OK;
}

}  // extern "C"

// The reference's own input generator, for pinning recon_sample_occ:
// out[0..k) = Rng(seed).sample_without_replacement(n, k) (rng.hpp:49-59).
extern "C" void recon_ref_sample(uint64_t seed, int32_t n, int32_t k, int32_t *out) {
    Rng rng(seed);
    const std::vector<int> v = rng.sample_without_replacement(n, k);
    for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
}

extern "C" recon_status recon_pipeline_batch_run_host(recon_ctx *c, const recon_pipeline_batch *pb) {
    return recon_pipeline_batch_run(c, pb);
}

extern "C" recon_status recon_min_cost_1d(recon_ctx *, int32_t ns, const int64_t *sources, int32_t nt,
                                          const int64_t *targets, int64_t *cost, int32_t *detail) {
    return guarded(detail, [&] {
        *cost = min_assignment_cost_1d(std::vector<long long>(sources, sources + ns),
                                       std::vector<long long>(targets, targets + nt));
    });
}

extern "C" recon_status recon_occupancy_dag_paths(recon_ctx *, int32_t, int32_t, int32_t P, const int64_t *off,
                                                  const int32_t *verts, int32_t *dag_src, int32_t *dag_dst,
                                                  int64_t dag_capacity, int64_t *dag_count, int32_t *detail) {
    return guarded(detail, [&] {
        std::vector<Path> paths(static_cast<size_t>(P));
        for (int32_t i = 0; i < P; ++i) paths[static_cast<size_t>(i)].vertices.assign(verts + off[i], verts + off[i + 1]);
        const MoveDag dag = occupancy_dag(paths);
        *dag_count = static_cast<int64_t>(dag.edges.size());
        if (*dag_count > dag_capacity) throw Failure{RECON_ERR_CAPACITY, RECON_D_NONE};
        for (size_t i = 0; i < dag.edges.size(); ++i) {
            dag_src[i] = dag.edges[i].first;
            dag_dst[i] = dag.edges[i].second;
        }
    });
}

// Validators: the reference's validate_solution / check_one_move_per_token /
// validate_batches on the decoded solution; failures map to recon_verdict
// bits by message (executor.cpp:38-219, batching.cpp:161-252).
namespace {

uint32_t bits_of(const ValidationReport &r, bool batch) {
    static const std::pair<const char *, uint32_t> sol[] = {
        {"leaves the grid", RECON_V_PATH_BOUNDS},
        {"two paths share source vertex", RECON_V_SHARED_SOURCE},
        {"two paths share target vertex", RECON_V_SHARED_TARGET},
        {"dependency dag has a cycle", RECON_V_DAG_CYCLE},
        {"stats.total_displacement does not equal", RECON_V_STATS_DISPLACEMENT},
        {"stats.displaced_tokens does not equal", RECON_V_STATS_DISPLACED},
        {"execution failed", RECON_V_EXECUTION},
        {"final configuration does not cover", RECON_V_TARGETS},
        {"schedule violates dag edge", RECON_V_DAG_ORDER},
        {"from an empty vertex", RECON_V_TOKEN_EMPTY},
        {"begins a second path", RECON_V_TOKEN_SECOND_PATH},
        {"matches no pending path edge", RECON_V_TOKEN_MATCH},
        {"edges missing from the schedule", RECON_V_TOKEN_MATCH},
    };
    static const std::pair<const char *, uint32_t> bat[] = {
        {"batched moves do not conserve", RECON_V_BATCH_CONSERVATION},
        {"more batches than elementary moves", RECON_V_BATCH_BOUND},
        {"is empty", RECON_V_BATCH_EMPTY},
        {"is not vertex-disjoint", RECON_V_BATCH_DISJOINT},
        {"violates the constraint set", RECON_V_BATCH_CONSTRAINT},
        {"moves a token from an empty vertex", RECON_V_BATCH_COLLISION},
        {"moves into a vertex occupied", RECON_V_BATCH_COLLISION},
        {"batched execution does not cover", RECON_V_BATCH_TARGETS},
        {"matches no pending path edge", RECON_V_BATCH_ORDER},
        {"edges missing from the schedule", RECON_V_BATCH_ORDER},
        {"batch order violates dag edge", RECON_V_BATCH_DAG},
    };
    uint32_t v = 0;
    for (const std::string &f : r.failures) {
        uint32_t b = 1u << 31;  // unmapped message
        if (batch) {
            for (const auto &[m, bit] : bat)
                if (f.find(m) != std::string::npos) {
                    b = bit;
                    break;
                }
        } else {
            for (const auto &[m, bit] : sol)
                if (f.find(m) != std::string::npos) {
                    b = bit;
                    break;
                }
        }
        v |= b;
    }
    return v;
}

uint32_t validate_ref(const recon_validate_batch *b, int i) {
    const int wpc = words_per_column(b->height);
    const Problem p = grid_problem(b->occ + static_cast<size_t>(i) * b->width * wpc, b->width, b->height, b->h_prime);
    const Geometry &g = p.geometry;
    const int np = b->path_count[i];
    const int32_t *ps = b->path_src + i * b->path_stride, *pt = b->path_dst + i * b->path_stride;
    PathSystem sys;
    bool oob = false;
    for (int k = 0; k < np; ++k) {
        if (!g.in_bounds(ps[k]) || !g.in_bounds(pt[k])) {
            Path q;
            q.vertices = {ps[k], pt[k]};
            sys.paths.push_back(q);
            oob = true;
        } else {
            sys.paths.push_back(one_bend_path(g, ps[k], pt[k]));
        }
    }
    MoveDag dag;
    dag.node_count = np;
    if (b->dag_mode == RECON_DAG_EXPLICIT) {
        for (int64_t e = b->dag_offset[i]; e < b->dag_offset[i + 1]; ++e) dag.add_edge(b->dag_a[e], b->dag_b[e]);
    } else if (b->dag_mode == RECON_DAG_OCCUPANCY && !oob) {
        dag = occupancy_dag(sys.paths);
    }
    std::vector<int> order(static_cast<size_t>(np));
    for (int k = 0; k < np; ++k) order[static_cast<size_t>(k)] = k;
    Solution sol;
    if (oob) {  // make_solution would walk out-of-grid vertices
        sol.path_system = sys;
        sol.dag = dag;
        sol.stats.displaced_tokens = np;
        sol.stats.total_displacement = 0;
    } else {
        sol = make_solution(sys, dag, order);
    }
    if (b->total_displacement) sol.stats.total_displacement = b->total_displacement[i];
    if (b->displaced) sol.stats.displaced_tokens = b->displaced[i];
    if (oob) return RECON_V_PATH_BOUNDS;  // a one-bend path needs in-grid endpoints; nothing else is evaluated
    uint32_t v = bits_of(validate_solution(p, sol), false);
    v |= bits_of(check_one_move_per_token(p, sol), false);
    if (b->move_batch) {
        const int32_t *mb = b->move_batch + i * b->move_stride;
        const int nb = b->batch_count[i];
        BatchSchedule bs;
        bs.batches.resize(static_cast<size_t>(std::max(nb, 0)));
        int64_t m = 0;
        for (const Path &q : sol.path_system.paths)
            for (size_t k = 0; k + 1 < q.vertices.size(); ++k, ++m) {
                const int32_t bi = mb[m];
                if (bi >= 0 && bi < nb) bs.batches[static_cast<size_t>(bi)].moves.push_back({q.vertices[k], q.vertices[k + 1]});
            }
        BatchOptions opt;
        opt.constraints.preset = b->preset == RECON_PRESET_COLUMN_DIRECTION ? ConstraintPreset::column_direction
                                                                            : ConstraintPreset::none;
        v |= bits_of(validate_batches(p, sol, bs, opt), true);
    }
    return v;
}

}  // namespace

extern "C" recon_status recon_validate_batch_run(recon_ctx *, const recon_validate_batch *b) {
    if (!b || !b->occ || !b->path_src || !b->path_dst || !b->path_count || !b->verdict) return RECON_ERR_ARGUMENT;
    parallel_for(b->count, [&](int i) { b->verdict[i] = validate_ref(b, i); });
    return RECON_OK;
}

extern "C" recon_status recon_validate_batch_run_host(recon_ctx *c, const recon_validate_batch *b) {
    return recon_validate_batch_run(c, b);
}

// Wire formats: the reference's own Solution / BatchSchedule content
// (make_solution's schedule, the dag, the paths; batches in ascending path id
// with tags from the first move) printed in the stock nlohmann dump(2) layout
// of io.cpp:81-164 (the reference's vendored json.hpp is not in its tree).
namespace {

struct JsonOut {
    std::string s;
    void sp(int k) { s.append(static_cast<size_t>(k), ' '); }
    void xy(const Geometry &g, int ind, Vertex v) {
        const Vec2 p = g.coords(v);
        s += "[\n";
        sp(ind + 2);
        s += std::to_string(p.x) + ",\n";
        sp(ind + 2);
        s += std::to_string(p.y) + "\n";
        sp(ind);
        s += "]";
    }
    void move(const Geometry &g, int ind, const ElementaryMove &m) {
        sp(ind);
        s += "[\n";
        sp(ind + 2);
        xy(g, ind + 2, m.from);
        s += ",\n";
        sp(ind + 2);
        xy(g, ind + 2, m.to);
        s += "\n";
        sp(ind);
        s += "]";
    }
};

recon_status json_out(const std::string &s, char *out, int64_t cap, int64_t *length) {
    *length = static_cast<int64_t>(s.size());
    if (cap < *length) return RECON_ERR_CAPACITY;
    std::memcpy(out, s.data(), s.size());
    return RECON_OK;
}

}  // namespace

extern "C" recon_status recon_solution_json(recon_ctx *, int32_t width, int32_t height, int32_t np,
                                            const int32_t *ps, const int32_t *pt, const int32_t *order, int64_t ne,
                                            const int32_t *ea, const int32_t *eb, int64_t displaced, int64_t total,
                                            char *out, int64_t cap, int64_t *length) {
    if (!length || width <= 0 || height <= 0 || np < 0 || ne < 0) return RECON_ERR_ARGUMENT;
    const Geometry g = Geometry::grid(width, height);
    PathSystem sys;
    for (int k = 0; k < np; ++k) sys.paths.push_back(one_bend_path(g, ps[k], pt[k]));
    MoveDag dag;
    dag.node_count = np;
    for (int64_t e = 0; e < ne; ++e) dag.add_edge(ea[e], eb[e]);
    std::vector<int> ord(static_cast<size_t>(np));
    for (int k = 0; k < np; ++k) ord[static_cast<size_t>(k)] = order ? order[k] : k;
    const Solution sol = make_solution(sys, dag, ord);
    JsonOut j;
    j.s = "{\n  \"moves\": ";
    if (sol.schedule.empty()) j.s += "[],\n";
    else {
        j.s += "[\n";
        for (size_t i = 0; i < sol.schedule.size(); ++i) {
            if (i) j.s += ",\n";
            j.move(g, 4, sol.schedule[i]);
        }
        j.s += "\n  ],\n";
    }
    j.s += "  \"dag_edges\": ";
    if (sol.dag.edges.empty()) j.s += "[],\n";
    else {
        j.s += "[\n";
        for (size_t i = 0; i < sol.dag.edges.size(); ++i) {
            if (i) j.s += ",\n";
            j.s += "    [\n      " + std::to_string(sol.dag.edges[i].first) + ",\n      " +
                   std::to_string(sol.dag.edges[i].second) + "\n    ]";
        }
        j.s += "\n  ],\n";
    }
    j.s += "  \"paths\": ";
    if (sol.path_system.paths.empty()) j.s += "[],\n";
    else {
        j.s += "[\n";
        for (size_t i = 0; i < sol.path_system.paths.size(); ++i) {
            if (i) j.s += ",\n";
            j.s += "    [\n";
            const Path &p = sol.path_system.paths[i];
            for (size_t k = 0; k < p.vertices.size(); ++k) {
                if (k) j.s += ",\n";
                j.sp(6);
                j.xy(g, 6, p.vertices[k]);
            }
            j.s += "\n    ]";
        }
        j.s += "\n  ],\n";
    }
    j.s += "  \"stats\": {\n    \"displaced_tokens\": " + std::to_string(displaced) +
           ",\n    \"total_displacement\": " + std::to_string(total) + "\n  }\n}\n";
    return json_out(j.s, out, cap, length);
}

extern "C" recon_status recon_solution_json_host(recon_ctx *c, int32_t width, int32_t height, int32_t np,
                                                 const int32_t *ps, const int32_t *pt, const int32_t *order,
                                                 int64_t ne, const int32_t *ea, const int32_t *eb, int64_t displaced,
                                                 int64_t total, char *out, int64_t cap, int64_t *length) {
    return recon_solution_json(c, width, height, np, ps, pt, order, ne, ea, eb, displaced, total, out, cap, length);
}

extern "C" recon_status recon_batch_schedule_json(recon_ctx *, int32_t width, int32_t height, int32_t np,
                                                  const int32_t *ps, const int32_t *pt, const int32_t *mb, int32_t nb,
                                                  int32_t preset, char *out, int64_t cap, int64_t *length) {
    if (!length || width <= 0 || height <= 0 || np < 0 || nb < 0) return RECON_ERR_ARGUMENT;
    const Geometry g = Geometry::grid(width, height);
    BatchSchedule bs;
    bs.batches.resize(static_cast<size_t>(nb));
    int64_t m = 0;
    for (int k = 0; k < np; ++k) {
        const Path p = one_bend_path(g, ps[k], pt[k]);
        for (size_t i = 0; i + 1 < p.vertices.size(); ++i, ++m)
            if (mb[m] >= 0 && mb[m] < nb) bs.batches[static_cast<size_t>(mb[m])].moves.push_back({p.vertices[i], p.vertices[i + 1]});
    }
    JsonOut j;
    j.s = "{\n  \"batches\": ";
    bool any = false;
    for (const Batch &b : bs.batches) {
        if (b.moves.empty()) continue;
        j.s += any ? ",\n" : "[\n";
        any = true;
        std::string ax = "null", dr = "null";
        if (preset == RECON_PRESET_COLUMN_DIRECTION) {
            const BatchDir d = move_dir(g, b.moves.front());
            ax = (d == BatchDir::up || d == BatchDir::down) ? "\"col\"" : "\"row\"";
            dr = d == BatchDir::up ? "\"up\"" : d == BatchDir::down ? "\"down\"" : d == BatchDir::left ? "\"left\"" : "\"right\"";
        }
        j.s += "    {\n      \"axis\": " + ax + ",\n      \"dir\": " + dr + ",\n      \"moves\": [\n";
        for (size_t i = 0; i < b.moves.size(); ++i) {
            if (i) j.s += ",\n";
            j.move(g, 8, b.moves[i]);
        }
        j.s += "\n      ]\n    }";
    }
    j.s += any ? "\n  ]\n}\n" : "[]\n}\n";
    return json_out(j.s, out, cap, length);
}

extern "C" recon_status recon_batch_schedule_json_host(recon_ctx *c, int32_t width, int32_t height, int32_t np,
                                                       const int32_t *ps, const int32_t *pt, const int32_t *mb,
                                                       int32_t nb, int32_t preset, char *out, int64_t cap,
                                                       int64_t *length) {
    return recon_batch_schedule_json(c, width, height, np, ps, pt, mb, nb, preset, out, cap, length);
}

// Loss simulation (SPEC.md [MODULE] sim; no reference code): the shared
// sequential restatement (oracle/sim_common.h) driving the compiled
// reference's own red_rec / bird / batch_moves.
#include "sim_common.h"

namespace {

recon_status ref_sim_solve(int batching, int solver, int preset, recon_grid_batch *g, int64_t ms, int32_t *mb,
                           int32_t *nb) {
    if (batching) {
        recon_pipeline_batch pb{*g, solver, preset, ms, mb, nb};
        return recon_pipeline_batch_run(nullptr, &pb);
    }
    return solver == 1 ? recon_bird_solve_batch(nullptr, g) : recon_redrec_solve_batch(nullptr, g);
}

}  // namespace

extern "C" recon_status recon_sim_run_host(recon_ctx *, const recon_sim_batch *b) {
    if (!b || !b->occ || !b->success || !b->cycles || !b->status || !b->n_nu || !b->n_alpha || !b->nb_nu ||
        !b->nb_alpha || !b->atoms_lost || !b->elapsed || b->width <= 0 || b->height <= 0 || b->h_prime <= 0 ||
        b->h_prime >= b->height)
        return RECON_ERR_ARGUMENT;
    parallel_for(b->count, [&](int i) { simc_trial(b, i, ref_sim_solve); });
    return RECON_OK;
}

// recon_pipeline_stats over host pointers (digest_cpu.h)
extern "C" recon_status recon_pipeline_stats(recon_ctx *, const recon_pipeline_batch *pb, recon_instance_stats *stats) {
    return recon_dg_stats(pb, stats);
}

// no device phases on the CPU checker
extern "C" recon_status recon_ctx_phase_times(recon_ctx *, float *ms, int32_t n) {
    for (int32_t i = 0; ms && i < n; ++i) ms[i] = 0.0f;
    return RECON_OK;
}

extern "C" recon_status recon_pipeline_schedule_runs(recon_ctx *, const recon_pipeline_batch *pb,
                                                     recon_schedule_runs *runs) {
    return recon_dg_runs(pb, runs);
}

// the pipeline into a temporary schedule, then its runs
extern "C" recon_status recon_pipeline_batch_run_host_runs(recon_ctx *c, const recon_pipeline_batch *pb,
                                                           recon_schedule_runs *runs) {
    if (!pb || !runs) return RECON_ERR_ARGUMENT;
    recon_pipeline_batch q = *pb;
    std::vector<int32_t> tmp;
    if (!q.move_batch) {
        tmp.resize(static_cast<size_t>(pb->grid.count) * static_cast<size_t>(pb->move_stride));
        q.move_batch = tmp.data();
    }
    recon_status st = recon_pipeline_batch_run_host(c, &q);
    if (st == RECON_OK) st = recon_dg_runs(&q, runs);
    return st;
}
