/*
 * raster_oracle.h — CPU oracle for the RASTER contraction + agglomeration
 * path. TEST INFRASTRUCTURE ONLY: this is the checker the GPU path is
 * compared against (tests/, __graft_entry__.smoke(), bench.py's CPU
 * baseline). The product library never links, loads or calls it.
 *
 * A plain-C restatement of the reference algorithm
 * (/root/reference/proj/include/raster, header-only C++20); every function
 * cites the reference lines it follows. Pinned against the reference's own
 * known-answer tests (tests/golden/kat_*.json) and against the reference
 * itself compiled from its headers (oracle/_ref, fixtures under
 * tests/golden/ref_*.npz made by tests/golden/make_golden.py).
 */
#ifndef RASTER_ORACLE_H_
#define RASTER_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_params {
    double precision;
    double x_min, x_max, y_min, y_max;
    uint64_t threshold;
    int32_t distance;
    int32_t metric; /* 0 chebyshev, 1 manhattan */
    uint64_t min_cluster_size;
} orc_params;

/* Canonical result: significant tiles sorted lexicographically, their counts
 * and cluster ids (-1 when the component was dropped by the mu filter). */
typedef struct orc_result {
    uint64_t n_ingested;
    uint64_t n_skipped;
    uint64_t n_distinct;   /* peak accumulator entries */
    uint64_t n_sig;
    int64_t* tx;
    int64_t* ty;
    uint64_t* count;
    int64_t* cluster_id;
    uint64_t n_components;
    uint64_t n_clusters;
} orc_result;

/* project_unchecked core.hpp:136-139 */
void orc_project(double x, double y, double scale, int64_t* tx, int64_t* ty);
/* cluster_sequential pipeline.hpp:92-126 (count-only mode, skip policy). */
int orc_cluster(const double* xy, uint64_t n, const orc_params* p, orc_result* out);
/* cluster_sequential with options: ORC_WINDOW_FIX = use_window_fix
 * (window_fix agglomerate.hpp:212-246 in place of prune, pipeline.hpp:103);
 * ORC_DEDUPE = Mode::retain_points with dedupe_points (accumulator.hpp:165-169,
 * 199-204): thresholds and counts on unique points per tile. */
#define ORC_WINDOW_FIX 1
#define ORC_DEDUPE 2
int orc_cluster_ex(const double* xy, uint64_t n, const orc_params* p, int flags,
                   orc_result* out);
/* agglomerate agglomerate.hpp:196-201 over caller tiles (any order). */
int orc_agglomerate(const int64_t* tx, const int64_t* ty, const uint64_t* count, uint64_t n,
                    const orc_params* p, orc_result* out);
/* Per-point labels from a result (RASTER' in input order). */
int orc_label_points(const double* xy, uint64_t n, const orc_params* p, const orc_result* r,
                     int32_t* labels);
void orc_free(orc_result* r);

#ifdef __cplusplus
}
#endif

#endif
