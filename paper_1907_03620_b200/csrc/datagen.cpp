// datagen.cpp — seeded synthetic workloads (see include/raster_datagen.h).
// Benchmark/test infrastructure: host-only, multithreaded, deterministic for
// any thread count.
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "../../include/raster_datagen.h"

namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;

inline uint64_t mix64(uint64_t z) {  // splitmix64 finaliser (bijective)
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

inline uint64_t rnd(uint64_t seed, uint64_t stream, uint64_t i) {
    const uint64_t key = mix64(seed ^ mix64(stream * 0x9e3779b97f4a7c15ull + 0x632be59bd9b4e019ull));
    return mix64(key + (i + 1) * 0x9e3779b97f4a7c15ull);
}

inline double unit(uint64_t u) { return (double)(u >> 11) * 0x1.0p-53; }  // [0, 1)

enum Stream : uint64_t {
    kCentreX = 1, kCentreY, kPointA, kPointB, kBlobX, kBlobY, kBlobA, kBlobB,
    kWalkX, kWalkY, kWalkAngle, kNoiseX, kNoiseY
};

inline void gauss(uint64_t seed, uint64_t sa, uint64_t sb, uint64_t i, double& z0, double& z1) {
    // Box-Muller on two independent words.
    const double u1 = 1.0 - unit(rnd(seed, sa, i));  // (0, 1]
    const double u2 = unit(rnd(seed, sb, i));
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = kTwoPi * u2;
    z0 = r * std::cos(th);
    z1 = r * std::sin(th);
}

template <typename F>
void parallel_for(uint64_t n, int threads, F&& f) {
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > n) threads = (int)(n ? n : 1);
    std::vector<std::thread> pool;
    const uint64_t share = n / threads, rem = n % threads;
    uint64_t begin = 0;
    for (int t = 0; t < threads; ++t) {
        const uint64_t len = share + ((uint64_t)t < rem ? 1 : 0);
        pool.emplace_back([&f, begin, len] { f(begin, begin + len); });
        begin += len;
    }
    for (auto& th : pool) th.join();
}

struct Feistel {
    uint32_t half_bits;
    uint64_t half_mask;
    uint64_t keys[4];
    uint64_t n;
    Feistel(uint64_t n_, uint64_t seed) : n(n_) {
        uint32_t bits = 2;
        while (bits < 64 && (1ull << bits) < n) ++bits;
        if (bits & 1) ++bits;
        half_bits = bits / 2;
        half_mask = (1ull << half_bits) - 1;
        for (int r = 0; r < 4; ++r) keys[r] = rnd(seed, 0xfe15 + r, 0);
    }
    uint64_t once(uint64_t v) const {
        uint64_t l = v >> half_bits, r = v & half_mask;
        for (int k = 0; k < 4; ++k) {
            const uint64_t nl = r;
            r = l ^ (mix64(r ^ keys[k]) & half_mask);
            l = nl;
        }
        return (l << half_bits) | r;
    }
    uint64_t operator()(uint64_t i) const {
        uint64_t v = once(i);
        while (v >= n) v = once(v);  // cycle walking keeps it a bijection of [0, n)
        return v;
    }
};

}  // namespace

extern "C" {

uint64_t rg_gen_count(const rg_gen_spec* s) {
    return s->n_clusters * s->points_per_cluster + s->blob_points +
           s->n_walks * s->walk_steps * s->points_per_step + s->n_noise;
}

int rg_generate(const rg_gen_spec* s, double* xy, int threads) {
    if (!s || !xy) return -1;
    const uint64_t seed = s->seed;
    const double w = s->x_hi - s->x_lo, h = s->y_hi - s->y_lo;
    uint64_t off = 0;

    // Gaussian clusters, points of one cluster consecutive.
    const uint64_t nc = s->n_clusters * s->points_per_cluster;
    if (nc) {
        const uint64_t ppc = s->points_per_cluster;
        parallel_for(nc, threads, [&](uint64_t b, uint64_t e) {
            for (uint64_t g = b; g < e; ++g) {
                const uint64_t c = g / ppc;
                const double cx = s->x_lo + unit(rnd(seed, kCentreX, c)) * w;
                const double cy = s->y_lo + unit(rnd(seed, kCentreY, c)) * h;
                double z0, z1;
                gauss(seed, kPointA, kPointB, g, z0, z1);
                xy[2 * (off + g)] = cx + s->sigma * z0;
                xy[2 * (off + g) + 1] = cy + s->sigma * z1;
            }
        });
        off += nc;
    }
    // Dense blob.
    if (s->blob_points) {
        const double bx = s->x_lo + unit(rnd(seed, kBlobX, 0)) * w;
        const double by = s->y_lo + unit(rnd(seed, kBlobY, 0)) * h;
        parallel_for(s->blob_points, threads, [&](uint64_t b, uint64_t e) {
            for (uint64_t g = b; g < e; ++g) {
                double z0, z1;
                gauss(seed, kBlobA, kBlobB, g, z0, z1);
                xy[2 * (off + g)] = bx + s->blob_sigma * z0;
                xy[2 * (off + g) + 1] = by + s->blob_sigma * z1;
            }
        });
        off += s->blob_points;
    }
    // Random walks: position 0 = uniform start, then steps of fixed length in
    // a uniform random direction; points_per_step identical copies per
    // position.
    if (s->n_walks && s->walk_steps && s->points_per_step) {
        const uint64_t per_walk = s->walk_steps * s->points_per_step;
        parallel_for(s->n_walks, threads, [&](uint64_t b, uint64_t e) {
            for (uint64_t wk = b; wk < e; ++wk) {
                double x = s->x_lo + unit(rnd(seed, kWalkX, wk)) * w;
                double y = s->y_lo + unit(rnd(seed, kWalkY, wk)) * h;
                double* o = xy + 2 * (off + wk * per_walk);
                for (uint64_t st = 0; st < s->walk_steps; ++st) {
                    if (st) {
                        const double th = kTwoPi * unit(rnd(seed, kWalkAngle, wk * s->walk_steps + st));
                        x += s->step * std::cos(th);
                        y += s->step * std::sin(th);
                    }
                    for (uint64_t c = 0; c < s->points_per_step; ++c) {
                        *o++ = x;
                        *o++ = y;
                    }
                }
            }
        });
        off += s->n_walks * per_walk;
    }
    // Uniform noise over the box.
    if (s->n_noise) {
        parallel_for(s->n_noise, threads, [&](uint64_t b, uint64_t e) {
            for (uint64_t g = b; g < e; ++g) {
                xy[2 * (off + g)] = s->x_lo + unit(rnd(seed, kNoiseX, g)) * w;
                xy[2 * (off + g) + 1] = s->y_lo + unit(rnd(seed, kNoiseY, g)) * h;
            }
        });
        off += s->n_noise;
    }
    return 0;
}

int rg_shuffle(const double* in, double* out, uint64_t n, uint64_t seed, int threads) {
    if (!in || !out) return -1;
    if (n == 0) return 0;
    const Feistel perm(n, seed);
    parallel_for(n, threads, [&](uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i) {
            const uint64_t j = perm(i);
            out[2 * i] = in[2 * j];
            out[2 * i + 1] = in[2 * j + 1];
        }
    });
    return 0;
}

}  // extern "C"
