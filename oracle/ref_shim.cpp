// ref_shim.cpp — extern "C" access to the REFERENCE implementation itself.
// TEST INFRASTRUCTURE ONLY (checker + CPU baseline; never part of the
// product). Compiled by oracle/build_ref.sh directly against the reference's
// own headers under /root/reference/proj/include (header-only C++20; no
// sources are copied into this repository) into oracle/_ref/libraster_ref.so.
//
// Calls exactly what a reference user calls: raster::cluster_sequential /
// cluster_parallel (pipeline.hpp:92-172), raster::agglomerate
// (agglomerate.hpp:196-201) and, for the point-retaining variant,
// cluster_sequential in Mode::retain_points.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "raster/raster.hpp"
#include "raster_oracle.h"

namespace {

thread_local std::string g_err;

raster::GridParams to_params(const orc_params* p) {
    raster::GridParams g;
    g.precision = p->precision;
    g.bounds = raster::Bounds{p->x_min, p->x_max, p->y_min, p->y_max};
    g.threshold = p->threshold;
    g.distance = p->distance;
    g.metric = p->metric ? raster::Metric::manhattan : raster::Metric::chebyshev;
    g.min_cluster_size = p->min_cluster_size;
    return g;
}

// Canonical flat form: all significant tiles (sorted) with counts and ids.
int flatten(const std::vector<std::pair<raster::Tile, std::uint64_t>>& sig,
            const raster::ClusterSet& cs, orc_result* out) {
    const std::uint64_t n = sig.size();
    out->n_sig = n;
    out->tx = (int64_t*)std::malloc((n ? n : 1) * 8);
    out->ty = (int64_t*)std::malloc((n ? n : 1) * 8);
    out->count = (uint64_t*)std::malloc((n ? n : 1) * 8);
    out->cluster_id = (int64_t*)std::malloc((n ? n : 1) * 8);
    std::vector<std::pair<raster::Tile, std::int64_t>> ids;
    for (const raster::Cluster& c : cs.clusters)
        for (const raster::Tile& t : c.tiles) ids.emplace_back(t, c.id);
    std::sort(ids.begin(), ids.end());
    std::size_t j = 0;
    for (std::uint64_t i = 0; i < n; ++i) {
        out->tx[i] = sig[i].first.x;
        out->ty[i] = sig[i].first.y;
        out->count[i] = sig[i].second;
        while (j < ids.size() && ids[j].first < sig[i].first) ++j;
        out->cluster_id[i] =
            (j < ids.size() && ids[j].first == sig[i].first) ? ids[j].second : -1;
    }
    out->n_clusters = cs.clusters.size();
    return 0;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// cluster_sequential / cluster_parallel over one span; canonical output.
// workers == 0: cluster_sequential; otherwise cluster_parallel with that many
// workers. Phase times (seconds) from PipelineStats pipeline.hpp:64-72.
int ref_cluster(const double* xy, uint64_t n, const orc_params* p, unsigned workers,
                orc_result* out, double* t_projection, double* t_clustering) {
    try {
        std::memset(out, 0, sizeof *out);
        const raster::GridParams params = to_params(p);
        std::span<const raster::Point> pts(reinterpret_cast<const raster::Point*>(xy), n);
        // Significant tiles with counts: the same accumulator the pipeline
        // builds (parity data only; the timed call is the pipeline below).
        raster::TileAccumulator acc(params);
        acc.ingest(pts);
        out->n_ingested = acc.total_ingested();
        out->n_skipped = acc.skipped();
        out->n_distinct = acc.entry_count();
        raster::SignificantTiles sig = acc.prune();
        std::vector<std::pair<raster::Tile, std::uint64_t>> flat;
        flat.reserve(sig.size());
        for (const auto& [t, s] : sig) flat.emplace_back(t, s.count);
        std::sort(flat.begin(), flat.end());

        raster::PipelineStats st;
        raster::ClusterSet cs =
            workers == 0
                ? raster::cluster_sequential(pts, params, false, &st)
                : raster::cluster_parallel(pts, params, raster::ParallelConfig{workers}, false,
                                           &st);
        if (t_projection) *t_projection = st.t_projection;
        if (t_clustering) *t_clustering = st.t_clustering;
        return flatten(flat, cs, out);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// cluster_sequential(pts, params, use_window_fix) pipeline.hpp:92-126 with
// options: flags & 1 = use_window_fix (window_fix agglomerate.hpp:212-246),
// flags & 2 = Mode::retain_points + dedupe_points.
int ref_cluster_flags(const double* xy, uint64_t n, const orc_params* p, int flags,
                      orc_result* out) {
    try {
        std::memset(out, 0, sizeof *out);
        raster::GridParams params = to_params(p);
        const bool wf = flags & 1;
        if (flags & 2) {
            params.mode = raster::Mode::retain_points;
            params.dedupe_points = true;
        }
        std::span<const raster::Point> pts(reinterpret_cast<const raster::Point*>(xy), n);
        raster::TileAccumulator acc(params);
        acc.ingest(pts);
        out->n_ingested = acc.total_ingested();
        out->n_skipped = acc.skipped();
        out->n_distinct = acc.entry_count();
        raster::SignificantTiles sig = wf ? raster::window_fix(acc, params) : acc.prune();
        std::vector<std::pair<raster::Tile, std::uint64_t>> flat;
        flat.reserve(sig.size());
        for (const auto& [t, s] : sig) flat.emplace_back(t, s.count);
        std::sort(flat.begin(), flat.end());
        raster::ClusterSet cs = raster::cluster_sequential(pts, params, wf, nullptr);
        return flatten(flat, cs, out);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Timing only: the reference pipeline, nothing else. Returns total seconds
// (PipelineStats::t_total) or a negative value on error.
double ref_time_pipeline(const double* xy, uint64_t n, const orc_params* p, unsigned workers,
                         uint64_t* n_clusters, double* t_projection, double* t_clustering) {
    try {
        const raster::GridParams params = to_params(p);
        std::span<const raster::Point> pts(reinterpret_cast<const raster::Point*>(xy), n);
        raster::PipelineStats st;
        raster::ClusterSet cs =
            workers == 0
                ? raster::cluster_sequential(pts, params, false, &st)
                : raster::cluster_parallel(pts, params, raster::ParallelConfig{workers}, false,
                                           &st);
        if (n_clusters) *n_clusters = cs.clusters.size();
        if (t_projection) *t_projection = st.t_projection;
        if (t_clustering) *t_clustering = st.t_clustering;
        return st.t_total;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

// ref_time_pipeline with a mode: retain != 0 runs Mode::retain_points
// (core.hpp:74; RASTER', every in-bounds point of a kept tile is stored,
// accumulator.hpp:131) — the reference's form of the point-retaining variant.
double ref_time_pipeline_mode(const double* xy, uint64_t n, const orc_params* p, unsigned workers,
                              int retain, uint64_t* n_clusters, double* t_projection,
                              double* t_clustering) {
    try {
        raster::GridParams params = to_params(p);
        if (retain) params.mode = raster::Mode::retain_points;
        std::span<const raster::Point> pts(reinterpret_cast<const raster::Point*>(xy), n);
        raster::PipelineStats st;
        raster::ClusterSet cs =
            workers == 0
                ? raster::cluster_sequential(pts, params, false, &st)
                : raster::cluster_parallel(pts, params, raster::ParallelConfig{workers}, false,
                                           &st);
        if (n_clusters) *n_clusters = cs.clusters.size();
        if (t_projection) *t_projection = st.t_projection;
        if (t_clustering) *t_clustering = st.t_clustering;
        return st.t_total;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

// agglomerate(SignificantTiles, params) over caller tiles.
int ref_agglomerate(const int64_t* tx, const int64_t* ty, const uint64_t* count, uint64_t n,
                    const orc_params* p, orc_result* out) {
    try {
        std::memset(out, 0, sizeof *out);
        const raster::GridParams params = to_params(p);
        raster::SignificantTiles sig;
        std::vector<std::pair<raster::Tile, std::uint64_t>> flat;
        for (uint64_t i = 0; i < n; ++i) {
            raster::Tile t{tx[i], ty[i]};
            sig[t].count = count ? count[i] : 0;
            flat.emplace_back(t, count ? count[i] : 0);
        }
        std::sort(flat.begin(), flat.end());
        raster::ClusterSet cs = raster::agglomerate(std::move(sig), params);
        return flatten(flat, cs, out);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Prime mode (RASTER'): cluster_sequential with Mode::retain_points. Writes
// every retained point as (cluster id, x, y) in the reference's output order
// (clusters by id, points sorted by point_less; write_cluster_points_csv
// io.hpp:208-222). Returns the number of rows, or -1.
int64_t ref_prime_points_ex(const double* xy, uint64_t n, const orc_params* p, int flags,
                            int64_t* cid, double* px, double* py, uint64_t cap) {
    try {
        raster::GridParams params = to_params(p);
        params.mode = raster::Mode::retain_points;
        params.dedupe_points = (flags & 2) != 0;
        std::span<const raster::Point> pts(reinterpret_cast<const raster::Point*>(xy), n);
        raster::ClusterSet cs = raster::cluster_sequential(pts, params, (flags & 1) != 0);
        uint64_t k = 0;
        for (const raster::Cluster& c : cs.clusters)
            for (const raster::Point& q : c.points) {
                if (k < cap) {
                    cid[k] = c.id;
                    px[k] = q.x;
                    py[k] = q.y;
                }
                ++k;
            }
        return (int64_t)k;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int64_t ref_prime_points(const double* xy, uint64_t n, const orc_params* p, int64_t* cid,
                         double* px, double* py, uint64_t cap) {
    return ref_prime_points_ex(xy, n, p, 0, cid, px, py, cap);
}

// Strict policy check: index-free message of the first OOB point, as thrown
// by TileAccumulator::ingest accumulator.hpp:123-125. Returns 1 if thrown.
int ref_strict_ingest(const double* xy, uint64_t n, const orc_params* p, char* msg,
                      uint64_t msg_len, uint64_t* ingested) {
    raster::GridParams params = to_params(p);
    params.oob_policy = raster::OobPolicy::strict;
    raster::TileAccumulator acc(params);
    std::span<const raster::Point> pts(reinterpret_cast<const raster::Point*>(xy), n);
    try {
        acc.ingest(pts);
        *ingested = acc.total_ingested();
        return 0;
    } catch (const raster::OutOfBoundsError& e) {
        std::snprintf(msg, msg_len, "%s", e.what());
        *ingested = acc.total_ingested();
        return 1;
    }
}

// Projection of single points (core.hpp:136-139) for the KATs.
void ref_project(double x, double y, double precision, int64_t* tx, int64_t* ty) {
    raster::GridParams g;
    g.precision = precision;
    const raster::Tile t = raster::project_unchecked(raster::Point{x, y}, g.scale());
    *tx = t.x;
    *ty = t.y;
}

void ref_free(orc_result* r) {
    std::free(r->tx);
    std::free(r->ty);
    std::free(r->count);
    std::free(r->cluster_id);
    std::memset(r, 0, sizeof *r);
}

}  // extern "C"
