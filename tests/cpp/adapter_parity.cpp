// adapter_parity.cpp — the C++ drop-in (include/raster_b200/gpu.hpp) against
// the reference library itself, over the reference's own types, in the style
// of the reference's acceptance suite (proj/tests/acceptance.cpp). Built by
// tests/cpp/build.sh against /root/reference/proj/include; run by
// tests/test_gpu_cpp.py on a B200. Exit code = number of failed checks.
#include <cstdio>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "raster/raster.hpp"
#include "raster_b200/gpu.hpp"

using namespace raster;

static int failures = 0;
#define CHECK(cond, what)                                              \
    do {                                                               \
        if (!(cond)) {                                                 \
            ++failures;                                                \
            std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
        }                                                              \
    } while (0)

static std::vector<Point> gaussian_clusters(std::size_t k, std::size_t per, double sigma,
                                            std::uint64_t seed, double noise_frac = 0.0) {
    std::mt19937_64 rng(seed);
    auto unit = [&] { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
    std::vector<Point> pts;
    for (std::size_t c = 0; c < k; ++c) {
        const double cx = -180.0 + 360.0 * unit(), cy = -90.0 + 180.0 * unit();
        for (std::size_t i = 0; i < per; ++i) {
            const double u1 = 1.0 - unit(), u2 = unit();
            const double r = std::sqrt(-2.0 * std::log(u1));
            pts.push_back({cx + sigma * r * std::cos(6.283185307179586 * u2),
                           cy + sigma * r * std::sin(6.283185307179586 * u2)});
        }
    }
    const auto noise = static_cast<std::size_t>(noise_frac * pts.size());
    for (std::size_t i = 0; i < noise; ++i) pts.push_back({-180.0 + 360.0 * unit(), -90.0 + 180.0 * unit()});
    return pts;
}

static std::vector<std::pair<Tile, std::uint64_t>> sorted_sig(const SignificantTiles& s) {
    std::vector<std::pair<Tile, std::uint64_t>> v;
    for (const auto& [t, st] : s) v.emplace_back(t, st.count);
    std::sort(v.begin(), v.end());
    return v;
}

int main() {
    // 1. cluster_sequential equality (ClusterSet ==, agglomerate.hpp:31) over
    //    the reference generator (datagen.hpp) and Gaussian data, 3 precisions.
    std::mt19937_64 rng(0xacce55);
    for (int round = 0; round < 12; ++round) {
        GridParams params;
        params.precision = std::vector<double>{2.0, 3.0, 3.5}[round % 3];
        params.threshold = 1 + rng() % 6;
        params.min_cluster_size = 1 + rng() % 5;
        std::vector<Point> pts;
        if (round % 2 == 0) {
            GenConfig gen;
            gen.cluster_count = 50 + rng() % 500;
            gen.seed = rng();
            gen.noise_fraction = 0.1;
            pts = generate(gen).points;
        } else {
            pts = gaussian_clusters(100 + rng() % 300, 400, 0.0005 * (1 + rng() % 8), rng(), 0.05);
        }
        PipelineStats s_ref, s_gpu;
        const ClusterSet a = raster::cluster_sequential(pts, params, false, &s_ref);
        const ClusterSet b = raster::gpu::cluster_sequential(pts, params, false, &s_gpu);
        CHECK(a == b, ("cluster_sequential round " + std::to_string(round)).c_str());
        CHECK(s_ref.n_points == s_gpu.n_points && s_ref.n_skipped == s_gpu.n_skipped &&
                  s_ref.peak_accumulator_entries == s_gpu.peak_accumulator_entries &&
                  s_ref.n_significant == s_gpu.n_significant,
              "PipelineStats counters");
    }
    // 2. Prime mode (RASTER'): Cluster::points equal, sorted by point_less.
    {
        GridParams params;
        params.precision = 3.0;
        params.mode = Mode::retain_points;
        const auto pts = gaussian_clusters(200, 500, 0.0005, 77, 0.1);
        CHECK(raster::cluster_sequential(pts, params) == raster::gpu::cluster_sequential(pts, params),
              "prime mode ClusterSet");
    }
    // 3. Accumulator: chunked + out-of-order ingestion, prune, accessors
    //    (acceptance.cpp criterion 6).
    {
        GenConfig gen;
        gen.cluster_count = 200;
        gen.seed = 0xc4a9;
        const auto pts = generate(gen).points;
        GridParams params;
        raster::TileAccumulator ref(params);
        ref.ingest(pts);
        const auto want = sorted_sig(ref.prune());
        std::mt19937_64 r2(0xc4aa);
        for (int round = 0; round < 5; ++round) {
            std::set<std::size_t> cut{0, pts.size()};
            for (int i = 0; i < 20; ++i) cut.insert(r2() % pts.size());
            std::vector<std::size_t> c(cut.begin(), cut.end());
            std::vector<std::span<const Point>> chunks;
            for (std::size_t i = 0; i + 1 < c.size(); ++i) chunks.emplace_back(pts.data() + c[i], c[i + 1] - c[i]);
            std::shuffle(chunks.begin(), chunks.end(), r2);
            raster::gpu::TileAccumulator acc(params);
            for (auto ch : chunks) acc.ingest(ch);
            CHECK(acc.total_ingested() == pts.size(), "total_ingested");
            const auto got = sorted_sig(acc.prune());
            CHECK(got == want, "chunked prune");
            CHECK(acc.entry_count() == 0, "prune consumes");
        }
        raster::TileAccumulator r(params);
        raster::gpu::TileAccumulator g(params);
        r.ingest(pts);
        g.ingest(pts);
        CHECK(r.entry_count() == g.entry_count(), "entry_count");
        std::size_t mism = 0;
        r.for_each_count([&](const Tile& t, std::uint64_t n) { mism += g.count_of(t) != n; });
        CHECK(mism == 0, "count_of");
    }
    // 4. agglomerate vs reference on random tile sets (criterion 2).
    {
        std::mt19937_64 r3(0x02ac1e);
        for (int round = 0; round < 40; ++round) {
            GridParams params;
            params.metric = (round % 2) ? Metric::manhattan : Metric::chebyshev;
            params.distance = 1 + (round / 2) % 2;
            params.min_cluster_size = 1 + round % 3;
            const std::size_t n = 100 + r3() % 4901;
            const auto extent = static_cast<std::int64_t>(std::sqrt(static_cast<double>(n) * 2.0));
            std::uniform_int_distribution<std::int64_t> coord(-extent, extent);
            SignificantTiles sig;
            while (sig.size() < n) sig[Tile{coord(r3), coord(r3)}].count = 5;
            CHECK(raster::agglomerate(sig, params) == raster::gpu::agglomerate(sig, params),
                  ("agglomerate round " + std::to_string(round)).c_str());
        }
    }
    // 5. Strict policy: same exception type and message.
    {
        GridParams params;
        params.precision = 2;
        params.oob_policy = OobPolicy::strict;
        const std::vector<Point> pts{{0.5, 0.5}, {500.0, 0.0}, {0.6, 0.6}};
        std::string a, b;
        try { raster::TileAccumulator(params).ingest(pts); } catch (const OutOfBoundsError& e) { a = e.what(); }
        try { raster::gpu::TileAccumulator(params).ingest(pts); } catch (const OutOfBoundsError& e) { b = e.what(); }
        CHECK(!a.empty() && a == b, "strict OutOfBoundsError message");
    }
    // 6. window_fix (agglomerate.hpp:212-246) and cluster_sequential with
    //    use_window_fix, against the reference; the accumulator copy and the
    //    const-ness of window_fix (test_agglomerate.cpp:255-277).
    {
        std::mt19937_64 r4(0x3f1c);
        for (int round = 0; round < 6; ++round) {
            GridParams params;
            params.precision = round % 2 ? 3.0 : 2.0;
            params.threshold = 2 + r4() % 6;
            params.min_cluster_size = 1 + r4() % 4;
            const auto pts = gaussian_clusters(100 + r4() % 200, 60, 0.004, r4(), 0.2);
            raster::TileAccumulator ra(params);
            raster::gpu::TileAccumulator ga(params);
            ra.ingest(pts);
            ga.ingest(pts);
            const std::size_t before = ga.entry_count();
            CHECK(sorted_sig(raster::window_fix(ra, params)) ==
                      sorted_sig(raster::gpu::window_fix(ga, params)),
                  ("window_fix round " + std::to_string(round)).c_str());
            CHECK(ga.entry_count() == before, "window_fix leaves the accumulator intact");
            raster::gpu::TileAccumulator copy = ga;
            CHECK(sorted_sig(copy.prune()) == sorted_sig(ga.prune()), "copied accumulator");
            PipelineStats s_ref, s_gpu;
            CHECK(raster::cluster_sequential(pts, params, true, &s_ref) ==
                      raster::gpu::cluster_sequential(pts, params, true, &s_gpu),
                  ("cluster_sequential window_fix round " + std::to_string(round)).c_str());
            CHECK(s_ref.n_significant == s_gpu.n_significant, "window_fix n_significant");
        }
    }
    // 7. Single pass over a PointSource (CountingSource io.hpp:63-84, as
    //    test_pipeline.cpp:68-82) through both the span fast path and the
    //    chunked path (a stream-only source, test_parallel.cpp:40-47), with
    //    prime mode on the chunked path.
    {
        struct StreamOnly : PointSource {
            explicit StreamOnly(std::span<const Point> p) : src(p) {}
            std::size_t read(std::span<Point> out) override { return src.read(out); }
            VectorSource src;
        };
        // > 4 Mi points: the stream-only source takes two pinned 4 Mi-point chunks
        const auto pts = gaussian_clusters(1100, 4000, 0.0005, 4242, 0.05);
        for (int prime = 0; prime < 2; ++prime) {
            GridParams params;
            params.precision = 3.0;
            if (prime) params.mode = Mode::retain_points;
            const ClusterSet want = raster::cluster_sequential(pts, params);
            VectorSource vs(pts);
            CountingSource cs1(vs);
            CHECK(raster::gpu::cluster_sequential(cs1, params) == want, "span source");
            CHECK(cs1.points_read() == pts.size(), "span source read once");
            StreamOnly so(pts);
            CountingSource cs2(so);
            CHECK(raster::gpu::cluster_sequential(cs2, params) == want, "stream-only source");
            CHECK(cs2.points_read() == pts.size(), "stream-only source read once");
        }
    }
    // 8. Config errors are ConfigError.
    {
        GridParams bad;
        bad.threshold = 0;
        bool thrown = false;
        try { raster::gpu::TileAccumulator acc(bad); } catch (const ConfigError&) { thrown = true; }
        CHECK(thrown, "ConfigError");
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
    return failures;
}
