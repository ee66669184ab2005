/*
 * raster_oracle.c — CPU oracle (TEST INFRASTRUCTURE ONLY; see
 * raster_oracle.h). Plain C99 restatement of the reference algorithm. All
 * references are to /root/reference/proj/include/raster/<file>:<line>.
 *
 * Floating point: the only arithmetic on coordinates is the IEEE double
 * product x * s followed by floor (core.hpp:136-139), and s = pow(10, p)
 * from the host libm (core.hpp:95). Compile without -ffast-math.
 */
#include "raster_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ core.hpp */

/* Bounds::contains core.hpp:33-35 (closed; NaN -> false) */
static int contains(const orc_params* p, double x, double y) {
    return x >= p->x_min && x <= p->x_max && y >= p->y_min && y <= p->y_max;
}

/* project_unchecked core.hpp:136-139 */
void orc_project(double x, double y, double scale, int64_t* tx, int64_t* ty) {
    *tx = (int64_t)floor(x * scale);
    *ty = (int64_t)floor(y * scale);
}

/* TileHash::mix core.hpp:57-62 */
static uint64_t mix(uint64_t v) {
    v += 0x9e3779b97f4a7c15ull;
    v = (v ^ (v >> 30)) * 0xbf58476d1ce4e5b9ull;
    v = (v ^ (v >> 27)) * 0x94d049bb133111ebull;
    return v ^ (v >> 31);
}

/* TileHash::operator() core.hpp:64-67 */
static uint64_t tile_hash(int64_t x, int64_t y) { return mix(mix((uint64_t)x) ^ (uint64_t)y); }

/* Tile operator<=> core.hpp:53 (lexicographic x then y) */
static int tile_cmp(int64_t ax, int64_t ay, int64_t bx, int64_t by) {
    if (ax != bx) return ax < bx ? -1 : 1;
    if (ay != by) return ay < by ? -1 : 1;
    return 0;
}

/* ------------------------------------------------------ accumulator.hpp */

typedef struct slot {
    int64_t x, y;
    uint64_t count; /* 0 = empty */
} slot;

typedef struct counts {
    slot* s;
    uint64_t cap, mask, used;
} counts;

static int counts_init(counts* c) {
    c->cap = 1024; /* kInitialCapacity accumulator.hpp:83 */
    c->mask = c->cap - 1;
    c->used = 0;
    c->s = (slot*)calloc(c->cap, sizeof(slot));
    return c->s ? 0 : -1;
}

/* TileCounts::grow accumulator.hpp:84-94 */
static int counts_grow(counts* c) {
    slot* old = c->s;
    const uint64_t old_cap = c->cap;
    c->cap *= 2;
    c->mask = c->cap - 1;
    c->s = (slot*)calloc(c->cap, sizeof(slot));
    if (!c->s) return -1;
    for (uint64_t i = 0; i < old_cap; ++i) {
        if (old[i].count == 0) continue;
        uint64_t j = tile_hash(old[i].x, old[i].y) & c->mask;
        while (c->s[j].count != 0) j = (j + 1) & c->mask;
        c->s[j] = old[i];
    }
    free(old);
    return 0;
}

/* TileCounts::add accumulator.hpp:33-50 */
static int counts_add(counts* c, int64_t x, int64_t y, uint64_t by) {
    if ((c->used + 1) * 10 >= c->cap * 7)
        if (counts_grow(c)) return -1;
    uint64_t i = tile_hash(x, y) & c->mask;
    for (;;) {
        slot* s = &c->s[i];
        if (s->count == 0) {
            s->x = x;
            s->y = y;
            s->count = by;
            ++c->used;
            return 0;
        }
        if (s->x == x && s->y == y) {
            s->count += by;
            return 0;
        }
        i = (i + 1) & c->mask;
    }
}

/* TileCounts::count_of accumulator.hpp:53-61, as a slot index (-1: absent) */
static int64_t counts_find(const counts* c, int64_t x, int64_t y) {
    uint64_t i = tile_hash(x, y) & c->mask;
    for (;;) {
        const slot* s = &c->s[i];
        if (s->count == 0) return -1;
        if (s->x == x && s->y == y) return (int64_t)i;
        i = (i + 1) & c->mask;
    }
}

static uint64_t counts_of(const counts* c, int64_t x, int64_t y) {
    const int64_t i = counts_find(c, x, y);
    return i < 0 ? 0 : c->s[i].count;
}

/* window_fix agglomerate.hpp:212-246: every occupied tile visits the four
 * 2x2 windows anchored at (x+ax, y+ay), ax, ay in {-1, 0} (:216-218); a
 * window whose total reaches the threshold (:225-226) marks its occupied
 * tiles (:227-229). The reference's anchors_seen set (:219) only skips
 * re-evaluating a window; the marked set is the same without it. */
static unsigned char* window_fix_marks(const counts* c, uint64_t threshold) {
    unsigned char* keep = (unsigned char*)calloc(c->cap, 1);
    if (!keep) return NULL;
    for (uint64_t i = 0; i < c->cap; ++i) {
        if (c->s[i].count == 0) continue;
        for (int ax = -1; ax <= 0; ++ax)
            for (int ay = -1; ay <= 0; ++ay) {
                const int64_t x0 = c->s[i].x + ax, y0 = c->s[i].y + ay;
                const int64_t wx[4] = {x0, x0 + 1, x0, x0 + 1};
                const int64_t wy[4] = {y0, y0, y0 + 1, y0 + 1};
                uint64_t total = 0;
                for (int w = 0; w < 4; ++w) total += counts_of(c, wx[w], wy[w]);
                if (total < threshold) continue;
                for (int w = 0; w < 4; ++w) {
                    const int64_t j = counts_find(c, wx[w], wy[w]);
                    if (j >= 0) keep[j] = 1;
                }
            }
    }
    return keep;
}

/* ------------------------------------------------------ agglomerate.hpp */

typedef struct tile {
    int64_t x, y;
    uint64_t count;
    int64_t cid;
    uint32_t group;
} tile;

static int cmp_tile(const void* a, const void* b) {
    const tile* p = (const tile*)a;
    const tile* q = (const tile*)b;
    return tile_cmp(p->x, p->y, q->x, q->y);
}

/* TileIndexMap agglomerate.hpp:83-116 */
typedef struct imap {
    int64_t* x;
    int64_t* y;
    uint32_t* idx;
    uint64_t mask;
} imap;

#define IMAP_EMPTY 0xffffffffu

static int imap_init(imap* m, uint64_t n) {
    uint64_t cap = 16;
    while (cap * 7 < n * 10) cap *= 2; /* :88 keep load factor under 70% */
    m->mask = cap - 1;
    m->x = (int64_t*)malloc(cap * sizeof(int64_t));
    m->y = (int64_t*)malloc(cap * sizeof(int64_t));
    m->idx = (uint32_t*)malloc(cap * sizeof(uint32_t));
    if (!m->x || !m->y || !m->idx) return -1;
    for (uint64_t i = 0; i < cap; ++i) m->idx[i] = IMAP_EMPTY;
    return 0;
}

static void imap_insert(imap* m, int64_t x, int64_t y, uint32_t index) { /* :94-98 */
    uint64_t i = tile_hash(x, y) & m->mask;
    while (m->idx[i] != IMAP_EMPTY) i = (i + 1) & m->mask;
    m->x[i] = x;
    m->y[i] = y;
    m->idx[i] = index;
}

static uint32_t imap_find(const imap* m, int64_t x, int64_t y) { /* :100-107 */
    uint64_t i = tile_hash(x, y) & m->mask;
    for (;;) {
        if (m->idx[i] == IMAP_EMPTY || (m->x[i] == x && m->y[i] == y)) return m->idx[i];
        i = (i + 1) & m->mask;
    }
}

static void imap_free(imap* m) {
    free(m->x);
    free(m->y);
    free(m->idx);
}

/* neighbor_offsets agglomerate.hpp:38-50 */
static int neighbor_offsets(const orc_params* p, int* dx, int* dy) {
    const int d = p->distance;
    int n = 0;
    for (int a = -d; a <= d; ++a)
        for (int b = -d; b <= d; ++b) {
            if (a == 0 && b == 0) continue;
            if (p->metric == 1 && abs(a) + abs(b) > d) continue;
            dx[n] = a;
            dy[n] = b;
            ++n;
        }
    return n;
}

typedef struct group {
    uint64_t first;  /* index (in sorted order) of the smallest tile */
    uint64_t size;
} group;

/* connected_components agglomerate.hpp:124-170 + agglomerate :196-201 +
 * finalize_clusters :175-191 over t[0..n) (any order on entry; sorted on
 * exit, with cid set). */
static int agglomerate_tiles(tile* t, uint64_t n, const orc_params* p, uint64_t* n_comp,
                             uint64_t* n_clusters) {
    *n_comp = *n_clusters = 0;
    if (n == 0) return 0;
    /* Sorting first does not change the partition (order invariance,
     * test_agglomerate.cpp:146-159); it lets group ids follow the canonical
     * order directly. */
    qsort(t, n, sizeof(tile), cmp_tile);
    const int maxoff = (2 * p->distance + 1) * (2 * p->distance + 1);
    int* dx = (int*)malloc(sizeof(int) * maxoff);
    int* dy = (int*)malloc(sizeof(int) * maxoff);
    const int noff = neighbor_offsets(p, dx, dy);
    imap m;
    if (imap_init(&m, n)) return -1;
    for (uint64_t i = 0; i < n; ++i) imap_insert(&m, t[i].x, t[i].y, (uint32_t)i); /* :135 */
    unsigned char* visited = (unsigned char*)calloc(n, 1);
    uint32_t* stack = (uint32_t*)malloc(n * sizeof(uint32_t));
    group* groups = (group*)malloc(n * sizeof(group));
    uint64_t ng = 0;
    for (uint64_t seed = 0; seed < n; ++seed) { /* :146-169 */
        if (visited[seed]) continue;
        visited[seed] = 1;
        uint64_t sp = 0, size = 1, first = seed;
        stack[sp++] = (uint32_t)seed;
        t[seed].group = (uint32_t)ng;
        while (sp) {
            const uint32_t u = stack[--sp];
            for (int o = 0; o < noff; ++o) {
                const uint32_t j = imap_find(&m, t[u].x + dx[o], t[u].y + dy[o]);
                if (j == IMAP_EMPTY || visited[j]) continue;
                visited[j] = 1;
                t[j].group = (uint32_t)ng;
                if (j < first) first = j;
                ++size;
                stack[sp++] = j;
            }
        }
        groups[ng].first = first;
        groups[ng].size = size;
        ++ng;
    }
    *n_comp = ng;
    /* erase_if(size < mu) :198-199; finalize: clusters ordered by smallest
     * tile :186-189, ids from 0 :189-190. Since t is sorted, "smallest tile"
     * is the smallest index, and groups were discovered in increasing order
     * of their smallest index (the DFS seeds sweep upward). */
    int64_t* gid = (int64_t*)malloc(ng * sizeof(int64_t));
    int64_t next = 0;
    for (uint64_t g = 0; g < ng; ++g)
        gid[g] = groups[g].size >= p->min_cluster_size ? next++ : -1;
    for (uint64_t i = 0; i < n; ++i) t[i].cid = gid[t[i].group];
    *n_clusters = (uint64_t)next;
    free(gid);
    free(groups);
    free(stack);
    free(visited);
    imap_free(&m);
    free(dx);
    free(dy);
    return 0;
}

static int fill_result(tile* t, uint64_t n, orc_result* out) {
    out->n_sig = n;
    out->tx = (int64_t*)malloc((n ? n : 1) * sizeof(int64_t));
    out->ty = (int64_t*)malloc((n ? n : 1) * sizeof(int64_t));
    out->count = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    out->cluster_id = (int64_t*)malloc((n ? n : 1) * sizeof(int64_t));
    if (!out->tx || !out->ty || !out->count || !out->cluster_id) return -1;
    for (uint64_t i = 0; i < n; ++i) {
        out->tx[i] = t[i].x;
        out->ty[i] = t[i].y;
        out->count[i] = t[i].count;
        out->cluster_id[i] = t[i].cid;
    }
    return 0;
}

/* dedupe (accumulator.hpp:199-204): unique points per tile, compared with
 * operator== on doubles (core.hpp:17; -0.0 == +0.0). */
typedef struct tpt {
    int64_t tx, ty;
    double x, y;
} tpt;

static int cmp_tpt(const void* a, const void* b) {
    const tpt* p = (const tpt*)a;
    const tpt* q = (const tpt*)b;
    const int t = tile_cmp(p->tx, p->ty, q->tx, q->ty);
    if (t) return t;
    if (p->x < q->x) return -1;
    if (p->x > q->x) return 1;
    if (p->y < q->y) return -1;
    if (p->y > q->y) return 1;
    return 0;
}

static int unique_counts(const double* xy, uint64_t n, const orc_params* p, double s,
                         counts* u) {
    tpt* a = (tpt*)malloc((n ? n : 1) * sizeof(tpt));
    if (!a) return -1;
    uint64_t m = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const double x = xy[2 * i], y = xy[2 * i + 1];
        if (!contains(p, x, y)) continue;
        orc_project(x, y, s, &a[m].tx, &a[m].ty);
        a[m].x = x;
        a[m].y = y;
        ++m;
    }
    qsort(a, m, sizeof(tpt), cmp_tpt);
    for (uint64_t i = 0; i < m; ++i) {
        if (i > 0 && a[i].tx == a[i - 1].tx && a[i].ty == a[i - 1].ty && a[i].x == a[i - 1].x &&
            a[i].y == a[i - 1].y)
            continue;
        if (counts_add(u, a[i].tx, a[i].ty, 1)) return -1;
    }
    free(a);
    return 0;
}

int orc_cluster(const double* xy, uint64_t n, const orc_params* p, orc_result* out) {
    return orc_cluster_ex(xy, n, p, 0, out);
}

int orc_cluster_ex(const double* xy, uint64_t n, const orc_params* p, int flags,
                   orc_result* out) {
    const int use_window_fix = flags & ORC_WINDOW_FIX;
    const int dedupe = flags & ORC_DEDUPE;
    memset(out, 0, sizeof *out);
    const double s = pow(10.0, p->precision); /* GridParams::scale core.hpp:95 */
    counts c;
    if (counts_init(&c)) return -1;
    /* TileAccumulator::ingest accumulator.hpp:120-134 (skip policy) */
    for (uint64_t i = 0; i < n; ++i) {
        const double x = xy[2 * i], y = xy[2 * i + 1];
        if (!contains(p, x, y)) {
            ++out->n_skipped;
            continue;
        }
        int64_t tx, ty;
        orc_project(x, y, s, &tx, &ty);
        if (counts_add(&c, tx, ty, 1)) return -1;
        ++out->n_ingested;
    }
    out->n_distinct = c.used;
    /* TileAccumulator::prune accumulator.hpp:160-174, or window_fix
     * (pipeline.hpp:103) */
    unsigned char* keep = NULL;
    if (use_window_fix && !(keep = window_fix_marks(&c, p->threshold))) return -1;
    /* dedupe: the threshold and the reported count use unique points
     * (accumulator.hpp:165-169); window_fix decides on raw counts (:225). */
    counts u;
    u.s = NULL;
    if (dedupe) {
        if (counts_init(&u) || unique_counts(xy, n, p, s, &u)) return -1;
        for (uint64_t i = 0; i < c.cap; ++i)
            if (c.s[i].count != 0) c.s[i].count = counts_of(&u, c.s[i].x, c.s[i].y);
        free(u.s);
    }
#define KEPT(i) (c.s[i].count != 0 && (keep ? keep[i] : c.s[i].count >= p->threshold))
    uint64_t ns = 0;
    for (uint64_t i = 0; i < c.cap; ++i)
        if (KEPT(i)) ++ns;
    tile* t = (tile*)malloc((ns ? ns : 1) * sizeof(tile));
    ns = 0;
    for (uint64_t i = 0; i < c.cap; ++i)
        if (KEPT(i)) {
            t[ns].x = c.s[i].x;
            t[ns].y = c.s[i].y;
            t[ns].count = c.s[i].count;
            ++ns;
        }
#undef KEPT
    free(keep);
    free(c.s);
    if (agglomerate_tiles(t, ns, p, &out->n_components, &out->n_clusters)) return -1;
    const int rc = fill_result(t, ns, out);
    free(t);
    return rc;
}

int orc_agglomerate(const int64_t* tx, const int64_t* ty, const uint64_t* count, uint64_t n,
                    const orc_params* p, orc_result* out) {
    memset(out, 0, sizeof *out);
    tile* t = (tile*)malloc((n ? n : 1) * sizeof(tile));
    for (uint64_t i = 0; i < n; ++i) {
        t[i].x = tx[i];
        t[i].y = ty[i];
        t[i].count = count ? count[i] : 0;
    }
    if (agglomerate_tiles(t, n, p, &out->n_components, &out->n_clusters)) return -1;
    const int rc = fill_result(t, n, out);
    free(t);
    return rc;
}

/* Label of a point = cluster id of its tile (prime mode keeps every
 * in-bounds point with its tile, accumulator.hpp:131; kept tiles hand their
 * points to their cluster, agglomerate.hpp:70-76,183). */
int orc_label_points(const double* xy, uint64_t n, const orc_params* p, const orc_result* r,
                     int32_t* labels) {
    const double s = pow(10.0, p->precision);
    for (uint64_t i = 0; i < n; ++i) {
        const double x = xy[2 * i], y = xy[2 * i + 1];
        labels[i] = -1;
        if (!contains(p, x, y)) continue;
        int64_t tx, ty;
        orc_project(x, y, s, &tx, &ty);
        uint64_t lo = 0, hi = r->n_sig;
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (tile_cmp(r->tx[mid], r->ty[mid], tx, ty) < 0)
                lo = mid + 1;
            else
                hi = mid;
        }
        if (lo < r->n_sig && r->tx[lo] == tx && r->ty[lo] == ty)
            labels[i] = (int32_t)r->cluster_id[lo];
    }
    return 0;
}

void orc_free(orc_result* r) {
    free(r->tx);
    free(r->ty);
    free(r->count);
    free(r->cluster_id);
    memset(r, 0, sizeof *r);
}
