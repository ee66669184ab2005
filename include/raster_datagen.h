/*
 * raster_datagen.h — seeded synthetic point generator for the BASELINE.json
 * workloads (benchmark/test infrastructure, not part of the clustering
 * path). The reference's own generator (datagen.hpp:195-228) only makes
 * uniform squares; the BASELINE configs need Gaussian clusters, noise, a
 * dense blob and random walks, so this is a new generator that keeps the
 * reference's portable-RNG discipline (datagen.hpp:24-41: randomness only
 * from 64-bit integer words, no std:: distributions).
 *
 * Coordinates: x = longitude in [-180, 180), y = latitude in [-90, 90)
 * (BASELINE.json's "[-90,90)x[-180,180)" read as (lat, lon); matches
 * Bounds::gps(), core.hpp:40-41).
 *
 * Randomness is counter-based (splitmix64 finaliser over (seed, stream,
 * index)), so any thread count produces identical bytes.
 * Output layout: interleaved float64 (x, y), generation order =
 * [clusters][blob][walks][noise].
 */
#ifndef RASTER_DATAGEN_H_
#define RASTER_DATAGEN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rg_gen_spec {
    uint64_t seed;
    uint64_t n_clusters;          /* Gaussian clusters                         */
    uint64_t points_per_cluster;
    double sigma;                 /* isotropic Gaussian sigma                  */
    uint64_t blob_points;         /* one dense Gaussian blob (0 = none)        */
    double blob_sigma;
    uint64_t n_walks;             /* random-walk chains                        */
    uint64_t walk_steps;          /* positions per walk                        */
    uint64_t points_per_step;     /* identical copies at each position         */
    double step;                  /* step length, uniform random direction     */
    uint64_t n_noise;             /* uniform points over the box               */
    double x_lo, x_hi, y_lo, y_hi; /* centre / start / noise box (half-open)   */
} rg_gen_spec;

uint64_t rg_gen_count(const rg_gen_spec* s);
/* Writes rg_gen_count(s) points (2 doubles each) into xy. threads <= 0: all
 * hardware threads. Returns 0 on success. */
int rg_generate(const rg_gen_spec* s, double* xy, int threads);
/* out[i] = in[perm(i)] for a seeded bijection perm of [0, n) (4-round
 * Feistel network with cycle walking). in and out must not overlap. */
int rg_shuffle(const double* in, double* out, uint64_t n, uint64_t seed, int threads);

#ifdef __cplusplus
}
#endif

#endif
