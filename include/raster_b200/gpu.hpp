// raster_b200/gpu.hpp — C++ drop-in for the reference's clustering path.
//
// Same signatures and semantics as the reference (header-only C++20 library
// /root/reference/proj/include/raster), over the reference's own types
// (raster::Point, Tile, GridParams, SignificantTiles, ClusterSet,
// PipelineStats), but every computation runs in the sm_100a library through
// the C-ABI in raster_gpu.h. A reference user switches by including this
// header and calling raster::gpu:: instead of raster::.
//
//   raster::TileAccumulator        accumulator.hpp:109-214  -> raster::gpu::TileAccumulator
//   raster::agglomerate            agglomerate.hpp:196-201  -> raster::gpu::agglomerate
//   raster::window_fix             agglomerate.hpp:212-246  -> raster::gpu::window_fix
//   raster::cluster_sequential     pipeline.hpp:92-126      -> raster::gpu::cluster_sequential
//
// Errors are the reference's exception types (errors.hpp:9-48): status codes
// map RG_ERR_CONFIG/UNSUPPORTED -> ConfigError, RG_ERR_OOB ->
// OutOfBoundsError (same message text as accumulator.hpp:124-125), anything
// else -> Error.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <optional>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "raster/accumulator.hpp"
#include "raster/agglomerate.hpp"
#include "raster/core.hpp"
#include "raster/errors.hpp"
#include "raster/io.hpp"
#include "raster/pipeline.hpp"
#include "raster_gpu.h"

static_assert(sizeof(raster::Point) == 2 * sizeof(double), "Point must be two packed doubles");

namespace raster::gpu {

inline rg_params to_rg(const GridParams& g) {
    rg_params p;
    rg_params_default(&p);
    p.precision = g.precision;
    p.x_min = g.bounds.x_min;
    p.x_max = g.bounds.x_max;
    p.y_min = g.bounds.y_min;
    p.y_max = g.bounds.y_max;
    p.threshold = g.threshold;
    p.distance = g.distance;
    p.metric = g.metric == Metric::manhattan ? RG_METRIC_MANHATTAN : RG_METRIC_CHEBYSHEV;
    p.min_cluster_size = g.min_cluster_size;
    p.mode = g.mode == Mode::retain_points ? RG_MODE_RETAIN_POINTS : RG_MODE_COUNT_ONLY;
    p.oob_policy = g.oob_policy == OobPolicy::strict ? RG_OOB_STRICT : RG_OOB_SKIP;
    p.dedupe_points = g.dedupe_points ? 1 : 0;
    return p;
}

[[noreturn]] inline void throw_status(rg_status s, const char* msg) {
    switch (s) {
        case RG_ERR_CONFIG:
        case RG_ERR_UNSUPPORTED: throw ConfigError(msg);
        case RG_ERR_OOB: throw OutOfBoundsError(msg);
        default: throw Error(msg);
    }
}

inline void check(rg_status s, const rg_ctx* ctx) {
    if (s != RG_OK) throw_status(s, rg_last_error(ctx));
}

namespace detail {

inline SignificantTiles significant_from(rg_ctx* ctx) {
    rg_stats st;
    check(rg_get_stats(ctx, &st), ctx);
    const std::uint64_t n = st.n_significant;
    std::vector<std::int64_t> tx(n), ty(n);
    std::vector<std::uint64_t> cnt(n);
    if (n) check(rg_get_significant(ctx, tx.data(), ty.data(), cnt.data(), nullptr, n, RG_MEM_HOST), ctx);
    SignificantTiles out;
    out.reserve(n);
    for (std::uint64_t i = 0; i < n; ++i) out[Tile{tx[i], ty[i]}].count = cnt[i];
    return out;
}

// finalize_clusters agglomerate.hpp:175-191 form from the canonical flat
// output (tiles sorted; ids by smallest tile).
inline ClusterSet clusters_from(rg_ctx* ctx) {
    rg_stats st;
    check(rg_get_stats(ctx, &st), ctx);
    const std::uint64_t n = st.n_significant, c = st.n_clusters;
    ClusterSet cs;
    cs.clusters.resize(c);
    for (std::uint64_t k = 0; k < c; ++k) cs.clusters[k].id = static_cast<std::int64_t>(k);
    if (n == 0 || c == 0) return cs;
    std::vector<std::int64_t> tx(n), ty(n), cid(n);
    check(rg_get_significant(ctx, tx.data(), ty.data(), nullptr, cid.data(), n, RG_MEM_HOST), ctx);
    for (std::uint64_t i = 0; i < n; ++i)
        if (cid[i] >= 0) cs.clusters[static_cast<std::size_t>(cid[i])].tiles.push_back(Tile{tx[i], ty[i]});
    return cs;
}

// RASTER' points: every in-bounds point of a kept cluster, grouped and
// sorted by point_less on the device (agglomerate.hpp:70-76,183,
// core.hpp:22-24).
inline void attach_points(rg_ctx* ctx, std::span<const Point> pts, ClusterSet& cs) {
    if (cs.clusters.empty() || pts.empty()) return;
    std::uint64_t m = 0, c = 0;
    check(rg_cluster_points(ctx, reinterpret_cast<const double*>(pts.data()), pts.size(),
                            RG_MEM_HOST, &m, &c),
          ctx);
    std::vector<Point> xy(m);
    std::vector<std::uint64_t> off(c + 1);
    check(rg_get_cluster_points(ctx, reinterpret_cast<double*>(xy.data()), m, off.data(),
                                RG_MEM_HOST),
          ctx);
    for (std::uint64_t k = 0; k < c && k < cs.clusters.size(); ++k)
        cs.clusters[k].points.assign(xy.begin() + off[k], xy.begin() + off[k + 1]);
}

}  // namespace detail

/// raster::TileAccumulator on the device (accumulator.hpp:109-214).
class TileAccumulator {
public:
    explicit TileAccumulator(GridParams params, int device = -1) : params_(std::move(params)) {
        params_.validate();  // accumulator.hpp:112
        const rg_params p = to_rg(params_);
        check(rg_create(&p, device, &ctx_), nullptr);
    }
    ~TileAccumulator() { rg_destroy(ctx_); }
    /// The reference's accumulator copy (test_agglomerate.cpp:268) on the device.
    TileAccumulator(const TileAccumulator& o) : params_(o.params_) {
        check(rg_clone(o.ctx_, &ctx_), nullptr);
    }
    TileAccumulator& operator=(const TileAccumulator& o) {
        if (this != &o) {
            TileAccumulator tmp(o);
            std::swap(params_, tmp.params_);
            std::swap(ctx_, tmp.ctx_);
        }
        return *this;
    }
    TileAccumulator(TileAccumulator&& o) noexcept
        : params_(std::move(o.params_)), ctx_(std::exchange(o.ctx_, nullptr)) {}
    TileAccumulator& operator=(TileAccumulator&& o) noexcept {
        std::swap(params_, o.params_);
        std::swap(ctx_, o.ctx_);
        return *this;
    }

    /// accumulator.hpp:117-134 (host span; staged through HBM).
    void ingest(std::span<const Point> pts) {
        check(rg_ingest(ctx_, reinterpret_cast<const double*>(pts.data()), pts.size(), RG_MEM_HOST), ctx_);
    }
    /// Zero-copy variant for points already resident in device memory.
    void ingest_device(const Point* pts, std::size_t n) {
        check(rg_ingest(ctx_, reinterpret_cast<const double*>(pts), n, RG_MEM_DEVICE), ctx_);
    }
    /// accumulator.hpp:137-154
    void merge(TileAccumulator&& other) { check(rg_merge(ctx_, other.ctx_), ctx_); }
    /// accumulator.hpp:156-174 — consumes the accumulator.
    SignificantTiles prune() {
        check(rg_prune(ctx_, nullptr), ctx_);
        return detail::significant_from(ctx_);
    }
    const GridParams& params() const noexcept { return params_; }
    std::size_t entry_count() const {
        std::uint64_t v = 0;
        check(rg_entry_count(ctx_, &v), ctx_);
        return static_cast<std::size_t>(v);
    }
    std::uint64_t count_of(const Tile& t) const {
        std::uint64_t v = 0;
        check(rg_count_of(ctx_, t.x, t.y, &v), ctx_);
        return v;
    }
    /// accumulator.hpp:188-191 over a snapshot (lexicographic order).
    template <typename F>
    void for_each_count(F&& fn) const {
        const std::size_t n = entry_count();
        std::vector<std::int64_t> tx(n), ty(n);
        std::vector<std::uint64_t> c(n);
        std::uint64_t got = 0;
        if (n) check(rg_export_counts(ctx_, tx.data(), ty.data(), c.data(), n, &got), ctx_);
        for (std::size_t i = 0; i < n; ++i) fn(Tile{tx[i], ty[i]}, c[i]);
    }
    std::uint64_t total_ingested() const {
        std::uint64_t v = 0;
        check(rg_total_ingested(ctx_, &v), ctx_);
        return v;
    }
    std::uint64_t skipped() const {
        std::uint64_t v = 0;
        check(rg_skipped(ctx_, &v), ctx_);
        return v;
    }
    rg_ctx* handle() noexcept { return ctx_; }

private:
    GridParams params_;
    rg_ctx* ctx_ = nullptr;
};

/// window_fix agglomerate.hpp:212-246 on the device. The accumulator is
/// left as it was (the kernel runs on a device copy).
inline SignificantTiles window_fix(const TileAccumulator& acc, const GridParams& params) {
    params.validate();
    TileAccumulator work(acc);
    check(rg_window_fix(work.handle(), nullptr), work.handle());
    return detail::significant_from(work.handle());
}

/// agglomerate agglomerate.hpp:196-201 on the device.
inline ClusterSet agglomerate(SignificantTiles sig, const GridParams& params) {
    params.validate();
    const rg_params p = to_rg(params);
    rg_ctx* ctx = nullptr;
    check(rg_create(&p, -1, &ctx), nullptr);
    struct Guard {
        rg_ctx* c;
        ~Guard() { rg_destroy(c); }
    } guard{ctx};
    std::vector<std::int64_t> tx, ty;
    std::vector<std::uint64_t> cnt;
    tx.reserve(sig.size());
    ty.reserve(sig.size());
    cnt.reserve(sig.size());
    for (const auto& [t, s] : sig) {
        tx.push_back(t.x);
        ty.push_back(t.y);
        cnt.push_back(s.count);
    }
    check(rg_load_significant(ctx, tx.data(), ty.data(), cnt.data(), tx.size(), RG_MEM_HOST), ctx);
    check(rg_agglomerate(ctx, nullptr), ctx);
    ClusterSet cs = detail::clusters_from(ctx);
    // Retained points travel with their tiles (agglomerate.hpp:70-76).
    if (params.mode == Mode::retain_points) {
        std::vector<std::pair<Tile, std::int64_t>> ids;
        for (const Cluster& c : cs.clusters)
            for (const Tile& t : c.tiles) ids.emplace_back(t, c.id);
        std::sort(ids.begin(), ids.end());
        for (auto& [t, s] : sig) {
            auto it = std::lower_bound(ids.begin(), ids.end(), std::make_pair(t, std::int64_t{-1}));
            if (it != ids.end() && it->first == t) {
                auto& dst = cs.clusters[static_cast<std::size_t>(it->second)].points;
                dst.insert(dst.end(), s.points.begin(), s.points.end());
            }
        }
        for (Cluster& c : cs.clusters) std::sort(c.points.begin(), c.points.end(), point_less);
    }
    return cs;
}

/// cluster_sequential pipeline.hpp:92-126 over a PointSource (single pass:
/// the whole-span fast path io.hpp:50-54, or 4 Mi-point chunks read into
/// pinned buffers while the previous chunk is copied and contracted).
inline ClusterSet cluster_sequential(PointSource& src, const GridParams& params,
                                     bool use_window_fix = false, PipelineStats* stats = nullptr) {
    params.validate();
    using Clock = std::chrono::steady_clock;
    const auto t0 = Clock::now();
    TileAccumulator acc(params);
    std::vector<Point> kept;  // retain mode needs the points again for labels
    std::span<const Point> all;
    if (auto span = src.take_full_span()) {
        acc.ingest(*span);
        all = *span;
    } else {
        // chunked source: the next read fills one pinned buffer while the
        // previous chunk is copied and contracted (rg_stream_*)
        rg_ctx* sctx = acc.handle();
        check(rg_stream_begin(sctx, std::uint64_t{1} << 22), sctx);
        while (true) {
            double* buf = nullptr;
            std::uint64_t cap = 0;
            check(rg_stream_buffer(sctx, &buf, &cap), sctx);
            std::span<Point> out(reinterpret_cast<Point*>(buf), static_cast<std::size_t>(cap));
            const std::size_t n = src.read(out);
            if (n == 0) break;
            if (params.mode == Mode::retain_points) kept.insert(kept.end(), out.begin(), out.begin() + n);
            const rg_status s = rg_stream_submit(sctx, n);
            if (s != RG_OK) {
                rg_stream_end(sctx);
                check(s, sctx);
            }
        }
        check(rg_stream_end(sctx), sctx);
        all = kept;
    }
    rg_ctx* ctx = acc.handle();
    rg_stats st;
    check(rg_get_stats(ctx, &st), ctx);
    const std::size_t peak = st.peak_accumulator_entries;
    const std::uint64_t ingested = st.n_ingested, skipped = st.n_skipped;
    // prune() or window_fix() (pipeline.hpp:103)
    check(use_window_fix ? rg_window_fix(ctx, nullptr) : rg_prune(ctx, nullptr), ctx);
    const double t_projection = std::chrono::duration<double>(Clock::now() - t0).count();
    const auto t1 = Clock::now();
    check(rg_agglomerate(ctx, nullptr), ctx);
    ClusterSet cs = detail::clusters_from(ctx);
    if (params.mode == Mode::retain_points) detail::attach_points(ctx, all, cs);
    check(rg_get_stats(ctx, &st), ctx);
    if (stats) {
        stats->t_projection = t_projection;
        stats->t_clustering = std::chrono::duration<double>(Clock::now() - t1).count();
        stats->t_total = std::chrono::duration<double>(Clock::now() - t0).count();
        stats->n_points = ingested + skipped;
        stats->n_skipped = skipped;
        stats->peak_accumulator_entries = peak;
        stats->n_significant = st.n_significant;
    }
    return cs;
}

inline ClusterSet cluster_sequential(std::span<const Point> pts, const GridParams& params,
                                     bool use_window_fix = false, PipelineStats* stats = nullptr) {
    VectorSource src(pts);
    return raster::gpu::cluster_sequential(src, params, use_window_fix, stats);
}

}  // namespace raster::gpu
