/* CPU oracle for the phfem hot path — TEST INFRASTRUCTURE (see
 * phfem_oracle.h for the pinning story).  Plain C11, built with
 * -ffp-contract=off so every expression rounds exactly like the reference's
 * C++ (SURVEY.md 8(a')).  Citations are file:line in proj/src of the
 * reference.
 */
#define _POSIX_C_SOURCE 200809L
#include "phfem_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "problems.h"

static _Thread_local char g_err[512];

const char* or_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

/* ------------------------------------------------------------------------ */
/* small vector algebra, geom.hpp:8-37                                      */

typedef struct { double x, y, z; } v3;

static inline v3 vsub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static inline v3 vadd(v3 a, v3 b) { v3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static inline v3 vmul(v3 a, double s) { v3 r = {a.x * s, a.y * s, a.z * s}; return r; }
static inline v3 vdiv(v3 a, double s) { v3 r = {a.x / s, a.y / s, a.z / s}; return r; }
static inline double vdot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline v3 vcross(v3 a, v3 b) {
    v3 r = {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
    return r;
}
static inline v3 node(const double* coords, int32_t n) {
    v3 r = {coords[3 * (int64_t)n], coords[3 * (int64_t)n + 1], coords[3 * (int64_t)n + 2]};
    return r;
}

/* local faces [abc],[acd],[adb],[dcb] (mesh.cpp:34-37, assembly.hpp:29) */
static const int kFaceVerts[4][3] = {{0, 1, 2}, {0, 2, 3}, {0, 3, 1}, {3, 2, 1}};
/* local edge order (connectivity.cpp:15-18) */
static const int kEdgeVerts[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

/* ------------------------------------------------------------------------ */
/* seeded inputs                                                            */

uint64_t or_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

double or_uniform(uint64_t seed, uint64_t idx) {
    return (double)(or_splitmix64(seed ^ idx) >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------------------ */
/* Kuhn meshes (not in the reference)                 */

static const int kKuhnPerm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
static const int kKuhnOdd[6] = {0, 1, 1, 0, 0, 1};

void or_kuhn_sizes(int nx, int ny, int nz, uint32_t mask, int64_t out[4]) {
    const int64_t per_plane[6] = {2ll * ny * nz, 2ll * ny * nz, 2ll * nx * nz,
                                  2ll * nx * nz, 2ll * nx * ny, 2ll * nx * ny};
    out[0] = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
    out[1] = 6ll * nx * ny * nz;
    out[2] = out[3] = 0;
    for (int p = 0; p < 6; ++p) {
        if (mask & (1u << p)) out[2] += per_plane[p];
        else out[3] += per_plane[p];
    }
}

void or_kuhn_mesh(int nx, int ny, int nz, double lx, double ly, double lz, double jitter,
                  uint64_t seed, uint32_t mask, double* coords, int32_t* tets, int32_t* db,
                  int32_t* nb) {
    const int64_t sx = nx + 1, sy = ny + 1;
    const double hx = lx / nx, hy = ly / ny, hz = lz / nz;
    for (int64_t k = 0; k <= nz; ++k)
        for (int64_t j = 0; j <= ny; ++j)
            for (int64_t i = 0; i <= nx; ++i) {
                const int64_t n = i + sx * (j + sy * k);
                double x = (lx * (double)i) / (double)nx;
                double y = (ly * (double)j) / (double)ny;
                double z = (lz * (double)k) / (double)nz;
                if (jitter != 0.0 && i > 0 && i < nx && j > 0 && j < ny && k > 0 && k < nz) {
                    x = x + ((2.0 * or_uniform(seed, 3 * (uint64_t)n) - 1.0) * jitter) * hx;
                    y = y + ((2.0 * or_uniform(seed, 3 * (uint64_t)n + 1) - 1.0) * jitter) * hy;
                    z = z + ((2.0 * or_uniform(seed, 3 * (uint64_t)n + 2) - 1.0) * jitter) * hz;
                }
                coords[3 * n] = x;
                coords[3 * n + 1] = y;
                coords[3 * n + 2] = z;
            }
    int64_t nd = 0, nnb = 0;
    for (int64_t k = 0; k < nz; ++k)
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t i = 0; i < nx; ++i) {
                const int64_t cell = i + nx * (j + ny * k);
                for (int p = 0; p < 6; ++p) {
                    int64_t idx[4][3];
                    int64_t a[3] = {i, j, k};
                    for (int d = 0; d < 3; ++d) idx[0][d] = a[d];
                    a[kKuhnPerm[p][0]] += 1;
                    for (int d = 0; d < 3; ++d) idx[1][d] = a[d];
                    a[kKuhnPerm[p][1]] += 1;
                    for (int d = 0; d < 3; ++d) idx[2][d] = a[d];
                    a[kKuhnPerm[p][2]] += 1;
                    for (int d = 0; d < 3; ++d) idx[3][d] = a[d];
                    if (kKuhnOdd[p]) {
                        for (int d = 0; d < 3; ++d) {
                            const int64_t tmp = idx[2][d];
                            idx[2][d] = idx[3][d];
                            idx[3][d] = tmp;
                        }
                    }
                    const int64_t t = 6 * cell + p;
                    for (int v = 0; v < 4; ++v)
                        tets[4 * t + v] = (int32_t)(idx[v][0] + sx * (idx[v][1] + sy * idx[v][2]));
                    for (int f = 0; f < 4; ++f) {
                        int plane = -1;
                        for (int d = 0; d < 3 && plane < 0; ++d) {
                            const int64_t c0 = idx[kFaceVerts[f][0]][d];
                            const int64_t c1 = idx[kFaceVerts[f][1]][d];
                            const int64_t c2 = idx[kFaceVerts[f][2]][d];
                            const int64_t nmax = d == 0 ? nx : d == 1 ? ny : nz;
                            if (c0 == c1 && c1 == c2 && (c0 == 0 || c0 == nmax))
                                plane = 2 * d + (c0 == 0 ? 0 : 1);
                        }
                        if (plane < 0) continue;
                        int32_t* dst = (mask & (1u << plane)) ? db + 3 * nd++ : nb + 3 * nnb++;
                        for (int v = 0; v < 3; ++v) dst[v] = tets[4 * t + kFaceVerts[f][v]];
                    }
                }
            }
}

/* ------------------------------------------------------------------------ */
/* open-addressing map uint64 -> int32 standing in for the reference's
 * unordered_map<uint64, EdgeId> (connectivity.hpp:25-30)                   */

typedef struct {
    uint64_t* keys;
    int32_t* vals;
    uint64_t mask;
} hmap;

static int hmap_init(hmap* m, int64_t n) {
    uint64_t cap = 16;
    while (cap < (uint64_t)(2 * n + 16)) cap <<= 1;
    m->keys = (uint64_t*)malloc(cap * sizeof(uint64_t));
    m->vals = (int32_t*)malloc(cap * sizeof(int32_t));
    if (!m->keys || !m->vals) return -1;
    memset(m->keys, 0xff, cap * sizeof(uint64_t));
    m->mask = cap - 1;
    return 0;
}

static void hmap_free(hmap* m) {
    free(m->keys);
    free(m->vals);
}

/* returns the existing value or inserts `val` and returns -1 - 0 */
static int32_t hmap_try_emplace(hmap* m, uint64_t key, int32_t val, int* inserted) {
    uint64_t h = or_splitmix64(key) & m->mask;
    for (;;) {
        if (m->keys[h] == key) {
            *inserted = 0;
            return m->vals[h];
        }
        if (m->keys[h] == UINT64_MAX) {
            m->keys[h] = key;
            m->vals[h] = val;
            *inserted = 1;
            return val;
        }
        h = (h + 1) & m->mask;
    }
}

static int32_t hmap_find(const hmap* m, uint64_t key) {
    uint64_t h = or_splitmix64(key) & m->mask;
    for (;;) {
        if (m->keys[h] == key) return m->vals[h];
        if (m->keys[h] == UINT64_MAX) return -1;
        h = (h + 1) & m->mask;
    }
}

typedef struct {
    hmap map;
    int64_t nc;
} edge_table;

/* EdgeTable::pair_to_edge (connectivity.hpp:25-30) */
static int32_t pair_to_edge(const edge_table* e, int32_t a, int32_t b) {
    if (a == b) return -1;
    if (a > b) { const int32_t t = a; a = b; b = t; }
    return hmap_find(&e->map, (uint64_t)a * (uint64_t)e->nc + (uint64_t)b);
}

/* num_edges, connectivity.cpp:22-37: first-occurrence numbering over the
 * slots 6t+k in local pair order, pairs sorted ascending. */
static int64_t build_edges(int64_t nc, int64_t ne, const int32_t* tets, edge_table* tab,
                           int32_t* edge_of_slot, int32_t* edge_nodes) {
    tab->nc = nc;
    if (hmap_init(&tab->map, 2 * ne + 8)) return -1;
    int64_t ned = 0;
    for (int64_t t = 0; t < ne; ++t)
        for (int k = 0; k < 6; ++k) {
            int32_t a = tets[4 * t + kEdgeVerts[k][0]], b = tets[4 * t + kEdgeVerts[k][1]];
            if (a > b) { const int32_t tmp = a; a = b; b = tmp; }
            int ins;
            const int32_t id = hmap_try_emplace(&tab->map, (uint64_t)a * (uint64_t)nc + (uint64_t)b,
                                                (int32_t)ned, &ins);
            if (ins) {
                if (edge_nodes) {
                    edge_nodes[2 * ned] = a;
                    edge_nodes[2 * ned + 1] = b;
                }
                ++ned;
            }
            if (edge_of_slot) edge_of_slot[6 * t + k] = id;
        }
    return ned;
}

int64_t or_num_edges(int64_t nc, int64_t ne, const int32_t* tets, int32_t* edge_of_slot,
                     int32_t* edge_nodes) {
    edge_table tab;
    const int64_t ned = build_edges(nc, ne, tets, &tab, edge_of_slot, edge_nodes);
    if (ned >= 0) hmap_free(&tab.map);
    return ned;
}

/* ------------------------------------------------------------------------ */
/* LSD radix sort of (uint64 key, int64 payload) by key; stable             */

static int radix_sort_u64(int64_t n, uint64_t* key, int64_t* val) {
    uint64_t* k2 = (uint64_t*)malloc((size_t)n * sizeof(uint64_t) + 8);
    int64_t* v2 = (int64_t*)malloc((size_t)n * sizeof(int64_t) + 8);
    if (!k2 || !v2) { free(k2); free(v2); return -1; }
    uint64_t maxk = 0;
    for (int64_t i = 0; i < n; ++i)
        if (key[i] > maxk) maxk = key[i];
    for (int shift = 0; shift < 64 && (shift == 0 || (maxk >> shift)); shift += 16) {
        int64_t cnt[65537];
        memset(cnt, 0, sizeof cnt);
        for (int64_t i = 0; i < n; ++i) cnt[((key[i] >> shift) & 0xffff) + 1]++;
        for (int d = 0; d < 65536; ++d) cnt[d + 1] += cnt[d];
        for (int64_t i = 0; i < n; ++i) {
            const int64_t pos = cnt[(key[i] >> shift) & 0xffff]++;
            k2[pos] = key[i];
            v2[pos] = val[i];
        }
        memcpy(key, k2, (size_t)n * sizeof(uint64_t));
        memcpy(val, v2, (size_t)n * sizeof(int64_t));
    }
    free(k2);
    free(v2);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* edge_pairs_to_elems, connectivity.cpp:46-70                              */

typedef struct {
    uint64_t* key; /* sorted */
    int64_t* elem;
    int64_t n;
    uint64_t ned;
} e2t_map;

static int build_e2t(int64_t ne, const int32_t* tets, const edge_table* edges, int64_t ned,
                     e2t_map* m) {
    m->n = 12 * ne;
    m->ned = (uint64_t)ned;
    m->key = (uint64_t*)malloc((size_t)m->n * sizeof(uint64_t) + 8);
    m->elem = (int64_t*)malloc((size_t)m->n * sizeof(int64_t) + 8);
    if (!m->key || !m->elem) return fail(2, "out of memory");
    int64_t i = 0;
    for (int64_t t = 0; t < ne; ++t)
        for (int k = 0; k < 4; ++k) {
            const int32_t x = tets[4 * t + kFaceVerts[k][0]];
            const int32_t y = tets[4 * t + kFaceVerts[k][1]];
            const int32_t z = tets[4 * t + kFaceVerts[k][2]];
            const uint64_t exy = (uint64_t)pair_to_edge(edges, x, y);
            const uint64_t eyz = (uint64_t)pair_to_edge(edges, y, z);
            const uint64_t ezx = (uint64_t)pair_to_edge(edges, z, x);
            m->key[i] = eyz * m->ned + exy; m->elem[i++] = t;
            m->key[i] = ezx * m->ned + eyz; m->elem[i++] = t;
            m->key[i] = exy * m->ned + ezx; m->elem[i++] = t;
        }
    if (radix_sort_u64(m->n, m->key, m->elem)) return fail(2, "out of memory");
    for (int64_t j = 1; j < m->n; ++j)
        if (m->key[j] == m->key[j - 1])
            return fail(2, "inconsistent mesh: elements %lld and %lld claim the same oriented face",
                        (long long)(m->elem[j - 1] + 1), (long long)(m->elem[j] + 1));
    return 0;
}

static void free_e2t(e2t_map* m) {
    free(m->key);
    free(m->elem);
}

/* EdgePairToElem::lookup, connectivity.cpp:39-44 */
static int64_t e2t_lookup(const e2t_map* m, int32_t from, int32_t to) {
    const uint64_t key = (uint64_t)from * m->ned + (uint64_t)to;
    int64_t lo = 0, hi = m->n;
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (m->key[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return (lo < m->n && m->key[lo] == key) ? m->elem[lo] : -1;
}

int or_edge_pairs_to_elems(int64_t nc, int64_t ne, const int32_t* tets, uint64_t* keys,
                           int32_t* elems) {
    edge_table edges;
    const int64_t ned = build_edges(nc, ne, tets, &edges, NULL, NULL);
    if (ned < 0) return fail(2, "out of memory");
    e2t_map m;
    int rc = build_e2t(ne, tets, &edges, ned, &m);
    if (!rc)
        for (int64_t i = 0; i < m.n; ++i) {
            keys[i] = m.key[i];
            elems[i] = (int32_t)m.elem[i];
        }
    free_e2t(&m);
    hmap_free(&edges.map);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* faces_up + full_face_table, connectivity.cpp:72-203                      */

/* face_area_and_normal, mesh.cpp:76-84 */
static int face_geom(const double* coords, const int32_t f[3], double* area, v3* unit) {
    const v3 p0 = node(coords, f[0]), p1 = node(coords, f[1]), p2 = node(coords, f[2]);
    const v3 n = vcross(vsub(p2, p0), vsub(p1, p0));
    const double len = sqrt(vdot(n, n));
    if (len == 0.0)
        return fail(2, "degenerate face with collinear nodes [%d %d %d]", f[0] + 1, f[1] + 1,
                    f[2] + 1);
    *area = 0.5 * len;
    if (unit) *unit = vdiv(n, len);
    return 0;
}

/* face_centroid, mesh.cpp:86-88 */
static v3 face_centroid(const double* coords, const int32_t f[3]) {
    return vdiv(vadd(vadd(node(coords, f[0]), node(coords, f[1])), node(coords, f[2])), 3.0);
}

typedef struct {
    uint64_t ab;
    int32_t c;
} trikey;

static trikey tri_key(const int32_t* f, int64_t nc) { /* connectivity.cpp:102-105 */
    int32_t s[3] = {f[0], f[1], f[2]};
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2 - i; ++j)
            if (s[j] > s[j + 1]) { const int32_t t = s[j]; s[j] = s[j + 1]; s[j + 1] = t; }
    trikey k = {(uint64_t)s[0] * (uint64_t)nc + (uint64_t)s[1], s[2]};
    return k;
}

static int same_cycle(const int32_t* a, const int32_t* b) { /* connectivity.cpp:107-111 */
    return (a[0] == b[0] && a[1] == b[1] && a[2] == b[2]) ||
           (a[0] == b[1] && a[1] == b[2] && a[2] == b[0]) ||
           (a[0] == b[2] && a[1] == b[0] && a[2] == b[1]);
}

typedef struct {
    uint64_t* ab;
    int32_t* c;
    int64_t* face;
    int64_t n;
    int64_t nc;
} face_index;

static int build_face_index(const int32_t* faces, int64_t nf, int64_t nc, face_index* ix) {
    ix->n = nf;
    ix->nc = nc;
    ix->ab = (uint64_t*)malloc((size_t)nf * sizeof(uint64_t) + 8);
    ix->c = (int32_t*)malloc((size_t)nf * sizeof(int32_t) + 8);
    ix->face = (int64_t*)malloc((size_t)nf * sizeof(int64_t) + 8);
    uint64_t* tmp = (uint64_t*)malloc((size_t)nf * sizeof(uint64_t) + 8);
    if (!ix->ab || !ix->c || !ix->face || !tmp) { free(tmp); return -1; }
    /* sort by (ab, c): stable LSD, c first then ab */
    for (int64_t f = 0; f < nf; ++f) {
        const trikey k = tri_key(faces + 3 * f, nc);
        tmp[f] = (uint64_t)(uint32_t)k.c;
        ix->face[f] = f;
    }
    if (radix_sort_u64(nf, tmp, ix->face)) { free(tmp); return -1; }
    for (int64_t i = 0; i < nf; ++i) tmp[i] = tri_key(faces + 3 * ix->face[i], nc).ab;
    if (radix_sort_u64(nf, tmp, ix->face)) { free(tmp); return -1; }
    for (int64_t i = 0; i < nf; ++i) {
        const trikey k = tri_key(faces + 3 * ix->face[i], nc);
        ix->ab[i] = k.ab;
        ix->c[i] = k.c;
    }
    free(tmp);
    return 0;
}

static void free_face_index(face_index* ix) {
    free(ix->ab);
    free(ix->c);
    free(ix->face);
}

static int64_t find_face(const face_index* ix, const int32_t* f) { /* connectivity.cpp:130-135 */
    const trikey k = tri_key(f, ix->nc);
    int64_t lo = 0, hi = ix->n;
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (ix->ab[mid] < k.ab || (ix->ab[mid] == k.ab && ix->c[mid] < k.c)) lo = mid + 1;
        else hi = mid;
    }
    return (lo < ix->n && ix->ab[lo] == k.ab && ix->c[lo] == k.c) ? ix->face[lo] : -1;
}

static void oriented_face(const int32_t* tet, int k, int32_t out[3]) {
    for (int v = 0; v < 3; ++v) out[v] = tet[kFaceVerts[k][v]];
}

int or_face_table(int64_t nc, int64_t ne, const int32_t* tets, const double* coords, int64_t nd,
                  const int32_t* db, int64_t nn, const int32_t* nb, int32_t* faces,
                  int32_t* face_of_slot, int8_t* sigma, int64_t* face_slots, uint8_t* face_class,
                  int32_t* mrow, double* area, int64_t counts[5]) {
    edge_table edges;
    const int64_t ned = build_edges(nc, ne, tets, &edges, NULL, NULL);
    if (ned < 0) return fail(2, "out of memory");
    e2t_map e2t;
    int rc = build_e2t(ne, tets, &edges, ned, &e2t);
    if (rc) { free_e2t(&e2t); hmap_free(&edges.map); return rc; }

    /* faces_up, connectivity.cpp:72-86 */
    int64_t nf = 0;
    for (int64_t s = 0; s < ne; ++s)
        for (int k = 0; k < 4; ++k) {
            int32_t f[3];
            oriented_face(tets + 4 * s, k, f);
            const int32_t exy = pair_to_edge(&edges, f[0], f[1]);
            const int32_t eyz = pair_to_edge(&edges, f[1], f[2]);
            const int64_t adj = e2t_lookup(&e2t, exy, eyz);
            if (adj < 0 || adj > s) {
                memcpy(faces + 3 * nf, f, sizeof f);
                ++nf;
            }
        }
    free_e2t(&e2t);
    hmap_free(&edges.map);

    /* full_face_table, connectivity.cpp:115-203 */
    face_index ix;
    if (build_face_index(faces, nf, nc, &ix)) return fail(2, "out of memory");
    for (int64_t f = 0; f < nf; ++f) face_slots[2 * f] = face_slots[2 * f + 1] = -1;
    for (int64_t t = 0; t < ne && !rc; ++t)
        for (int k = 0; k < 4; ++k) {
            const int64_t slot = 4 * t + k;
            int32_t of[3];
            oriented_face(tets + 4 * t, k, of);
            const int64_t f = find_face(&ix, of);
            if (f < 0) {
                rc = fail(2, "inconsistent mesh: face [%d %d %d] of element %lld matches no unique face",
                          of[0] + 1, of[1] + 1, of[2] + 1, (long long)(t + 1));
                break;
            }
            face_of_slot[slot] = (int32_t)f;
            sigma[slot] = same_cycle(of, faces + 3 * f) ? 1 : -1;
            if (face_slots[2 * f] < 0) face_slots[2 * f] = slot;
            else if (face_slots[2 * f + 1] < 0) face_slots[2 * f + 1] = slot;
            else {
                rc = fail(2, "inconsistent mesh: face [%d %d %d] is shared by more than two elements",
                          faces[3 * f] + 1, faces[3 * f + 1] + 1, faces[3 * f + 2] + 1);
                break;
            }
        }
    if (rc) { free_face_index(&ix); return rc; }

    /* classification, connectivity.cpp:156-175 */
    uint8_t* classified = (uint8_t*)calloc((size_t)nf + 1, 1);
    for (int64_t f = 0; f < nf; ++f) face_class[f] = 0;
    for (int pass = 0; pass < 2 && !rc; ++pass) {
        const int32_t* list = pass == 0 ? db : nb;
        const int64_t cnt = pass == 0 ? nd : nn;
        const char* what = pass == 0 ? "Dirichlet" : "Neumann";
        for (int64_t i = 0; i < cnt; ++i) {
            const int32_t* bf = list + 3 * i;
            const int64_t f = find_face(&ix, bf);
            if (f < 0) {
                rc = fail(2, "inconsistent mesh: %s face [%d %d %d] matches no element face", what,
                          bf[0] + 1, bf[1] + 1, bf[2] + 1);
                break;
            }
            if (classified[f]) {
                rc = fail(2, "inconsistent mesh: boundary face [%d %d %d] listed twice", bf[0] + 1,
                          bf[1] + 1, bf[2] + 1);
                break;
            }
            if (face_slots[2 * f + 1] >= 0) {
                rc = fail(2, "inconsistent mesh: %s face [%d %d %d] is interior", what, bf[0] + 1,
                          bf[1] + 1, bf[2] + 1);
                break;
            }
            classified[f] = 1;
            face_class[f] = (uint8_t)(pass + 1);
        }
    }
    free_face_index(&ix);

    /* areas, checks, multiplier rows, connectivity.cpp:177-201 */
    int64_t nint = 0, ndir = 0, nneu = 0;
    int32_t next_row = 0;
    for (int64_t f = 0; f < nf && !rc; ++f) {
        rc = face_geom(coords, faces + 3 * f, &area[f], NULL);
        if (rc) break;
        const int32_t* tri = faces + 3 * f;
        if (face_slots[2 * f + 1] < 0) {
            if (!classified[f]) {
                rc = fail(2, "inconsistent mesh: boundary face [%d %d %d] is in neither the Dirichlet nor the Neumann list",
                          tri[0] + 1, tri[1] + 1, tri[2] + 1);
                break;
            }
            if (sigma[face_slots[2 * f]] != 1) {
                rc = fail(2, "inconsistent mesh: stored orientation of boundary face [%d %d %d] does not match its element",
                          tri[0] + 1, tri[1] + 1, tri[2] + 1);
                break;
            }
        } else if (sigma[face_slots[2 * f]] + sigma[face_slots[2 * f + 1]] != 0) {
            rc = fail(2, "inconsistent mesh: interior face [%d %d %d] lacks the +1/-1 orientation pairing",
                      tri[0] + 1, tri[1] + 1, tri[2] + 1);
            break;
        }
        if (face_class[f] == 0) ++nint;
        else if (face_class[f] == 1) ++ndir;
        else ++nneu;
        mrow[f] = face_class[f] != 2 ? next_row++ : -1;
    }
    free(classified);
    if (rc) return rc;
    counts[0] = nf;
    counts[1] = nint;
    counts[2] = ndir;
    counts[3] = nneu;
    counts[4] = nint + ndir;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* red_refine + refine_boundary_faces, refine.cpp:16-96                     */

static int refine_faces(const int32_t* in, int64_t nf, const edge_table* edges,
                        const int32_t* midpoint, int32_t* out) {
    for (int64_t f = 0; f < nf; ++f) {
        const int32_t n1 = in[3 * f], n2 = in[3 * f + 1], n3 = in[3 * f + 2];
        const int32_t pr[3][2] = {{n1, n2}, {n2, n3}, {n1, n3}};
        int32_t m[3];
        for (int q = 0; q < 3; ++q) {
            const int32_t e = pair_to_edge(edges, pr[q][0], pr[q][1]);
            if (e < 0 || midpoint[e] < 0)
                return fail(2, "inconsistent mesh: boundary face edge (%d,%d) is not an element edge",
                            pr[q][0] + 1, pr[q][1] + 1);
            m[q] = midpoint[e];
        }
        const int32_t m12 = m[0], m23 = m[1], m13 = m[2];
        int32_t* o = out + 3 * f;
        o[0] = n1; o[1] = m12; o[2] = m13;
        o = out + 3 * (nf + 3 * f);
        o[0] = n2; o[1] = m23; o[2] = m12;
        o[3] = n3; o[4] = m13; o[5] = m23;
        o[6] = m12; o[7] = m23; o[8] = m13;
    }
    return 0;
}

int or_refine(int64_t nc, int64_t ne, const double* coords, const int32_t* tets, int64_t nd,
              const int32_t* db, int64_t nn, const int32_t* nb, double* coords_out,
              int32_t* tets_out, int32_t* db_out, int32_t* nb_out, int32_t* midpoint_node,
              int32_t* centroid_node) {
    edge_table edges;
    int32_t* eos = (int32_t*)malloc((size_t)(6 * ne + 1) * sizeof(int32_t));
    if (!eos) return fail(2, "out of memory");
    const int64_t ned = build_edges(nc, ne, tets, &edges, eos, NULL);
    if (ned < 0) { free(eos); return fail(2, "out of memory"); }
    int32_t* mid = (int32_t*)malloc((size_t)(ned + 1) * sizeof(int32_t));
    int32_t* cen = (int32_t*)malloc((size_t)(ne + 1) * sizeof(int32_t));
    for (int64_t e = 0; e < ned; ++e) mid[e] = -1;
    memcpy(coords_out, coords, (size_t)(3 * nc) * sizeof(double));
    int64_t next = nc;
    /* new nodes in first-occurrence order (refine.cpp:29-46) */
    for (int64_t t = 0; t < ne; ++t) {
        const int32_t* e = tets + 4 * t;
        const v3 ct = vdiv(vadd(vadd(vadd(node(coords, e[0]), node(coords, e[1])), node(coords, e[2])),
                                node(coords, e[3])),
                           4.0);
        cen[t] = (int32_t)next;
        coords_out[3 * next] = ct.x;
        coords_out[3 * next + 1] = ct.y;
        coords_out[3 * next + 2] = ct.z;
        ++next;
        for (int k = 0; k < 6; ++k) {
            const int32_t ed = eos[6 * t + k];
            if (mid[ed] < 0) {
                mid[ed] = (int32_t)next;
                const v3 pm = vdiv(vadd(node(coords, e[kEdgeVerts[k][0]]), node(coords, e[kEdgeVerts[k][1]])), 2.0);
                coords_out[3 * next] = pm.x;
                coords_out[3 * next + 1] = pm.y;
                coords_out[3 * next + 2] = pm.z;
                ++next;
            }
        }
    }
    /* children, refine.cpp:52-69 */
    for (int64_t t = 0; t < ne; ++t) {
        const int32_t* e = tets + 4 * t;
        const int32_t i = e[0], j = e[1], k = e[2], l = e[3];
        const int32_t ij = mid[eos[6 * t + 0]], ik = mid[eos[6 * t + 1]], il = mid[eos[6 * t + 2]];
        const int32_t jk = mid[eos[6 * t + 3]], jl = mid[eos[6 * t + 4]], kl = mid[eos[6 * t + 5]];
        const int32_t cn = cen[t];
        const int32_t ch[12][4] = {{i, ij, ik, il},  {j, jk, ij, jl},  {k, ik, jk, kl},  {l, kl, jl, il},
                                   {ij, ik, il, cn}, {jk, ij, jl, cn}, {ik, jk, kl, cn}, {kl, jl, il, cn},
                                   {ij, jk, ik, cn}, {ik, kl, il, cn}, {ij, il, jl, cn}, {kl, jk, jl, cn}};
        memcpy(tets_out + 4 * t, ch[0], 4 * sizeof(int32_t));
        for (int q = 1; q < 12; ++q) memcpy(tets_out + 4 * (ne + 11 * t + (q - 1)), ch[q], 4 * sizeof(int32_t));
    }
    int rc = 0;
    if (db_out) rc = refine_faces(db, nd, &edges, mid, db_out);
    if (!rc && nb_out) rc = refine_faces(nb, nn, &edges, mid, nb_out);
    if (midpoint_node) memcpy(midpoint_node, mid, (size_t)ned * sizeof(int32_t));
    if (centroid_node) memcpy(centroid_node, cen, (size_t)ne * sizeof(int32_t));
    free(mid);
    free(cen);
    free(eos);
    hmap_free(&edges.map);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* quadrature, quadrature.cpp:9-62                                          */

static void gauss_legendre(int n, double* x, double* w) {
    for (int i = 0; i < n; ++i) {
        double t = cos(M_PI * (i + 0.75) / (n + 0.5));
        double dp = 0.0;
        for (int iter = 0; iter < 100; ++iter) {
            double p0 = 1.0, p1 = t;
            for (int k = 2; k <= n; ++k) {
                const double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (t * p1 - p0) / (t * t - 1.0);
            const double dt = p1 / dp;
            t -= dt;
            if (fabs(dt) < 1e-15) break;
        }
        x[n - 1 - i] = 0.5 * (1.0 + t);
        w[n - 1 - i] = 1.0 / ((1.0 - t * t) * dp * dp);
    }
}

int or_tet_rule(int degree, double* lambda, double* w) {
    const int n = (degree + 3 + 1) / 2;
    double gx[16], gw[16];
    gauss_legendre(n, gx, gw);
    int q = 0;
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b)
            for (int c = 0; c < n; ++c) {
                const double u = gx[a], v = gx[b], ww = gx[c];
                const double x = u;
                const double y = v * (1.0 - u);
                const double z = ww * (1.0 - u) * (1.0 - v);
                const double jac = (1.0 - u) * (1.0 - u) * (1.0 - v);
                lambda[4 * q] = 1.0 - x - y - z;
                lambda[4 * q + 1] = x;
                lambda[4 * q + 2] = y;
                lambda[4 * q + 3] = z;
                w[q] = 6.0 * gw[a] * gw[b] * gw[c] * jac;
                ++q;
            }
    return q;
}

/* ------------------------------------------------------------------------ */
/* element matrices, assembly.cpp:7-33 (+ coefficient extension)            */

typedef struct {
    double k[4][4], m[4][4], a[4][4];
    double volume;
    v3 g[4];
} local_mats;

static void coef_of(const or_problem* p, int64_t t, double A[3]) {
    if (p && p->a_diag) {
        A[0] = p->a_diag[3 * t]; A[1] = p->a_diag[3 * t + 1]; A[2] = p->a_diag[3 * t + 2];
    } else if (p && p->a_elem) {
        A[0] = A[1] = A[2] = p->a_elem[t];
    } else {
        A[0] = A[1] = A[2] = 1.0;
    }
}

static int local_stiffness_mass(const double* coords, const int32_t* tet, int64_t t,
                                const double A[3], double c, local_mats* out) {
    const v3 p0 = node(coords, tet[0]);
    const v3 d1 = vsub(node(coords, tet[1]), p0);
    const v3 d2 = vsub(node(coords, tet[2]), p0);
    const v3 d3 = vsub(node(coords, tet[3]), p0);
    const double det = vdot(vcross(d1, d2), d3);
    if (det == 0.0) return fail(2, "degenerate element %lld (zero volume)", (long long)(t + 1));
    out->volume = fabs(det) / 6.0;
    out->g[1] = vdiv(vcross(d2, d3), det);
    out->g[2] = vdiv(vcross(d3, d1), det);
    out->g[3] = vdiv(vcross(d1, d2), det);
    out->g[0] = vmul(vadd(vadd(out->g[1], out->g[2]), out->g[3]), -1.0);
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            const v3 gi = out->g[i], gj = out->g[j];
            /* A = I: A0*(gx gx') + ... == dot(gi, gj) exactly */
            const double d = A[0] * (gi.x * gj.x) + A[1] * (gi.y * gj.y) + A[2] * (gi.z * gj.z);
            out->k[i][j] = out->volume * d;
            out->m[i][j] = out->volume / 20.0 * (i == j ? 2.0 : 1.0);
            out->a[i][j] = out->k[i][j] + c * out->m[i][j]; /* mat4_add, geom.hpp:34-39 */
        }
    return 0;
}

/* Mat4Lu, geom.hpp:48-87 */
typedef struct {
    double lu[4][4];
    int perm[4];
    int singular;
} lu4;

static void lu_factor(const double a[4][4], lu4* f) {
    memcpy(f->lu, a, sizeof f->lu);
    f->singular = 0;
    for (int i = 0; i < 4; ++i) f->perm[i] = i;
    for (int col = 0; col < 4; ++col) {
        int piv = col;
        double best = fabs(f->lu[col][col]);
        for (int r = col + 1; r < 4; ++r) {
            const double v = fabs(f->lu[r][col]);
            if (v > best) { best = v; piv = r; }
        }
        if (best == 0.0) { f->singular = 1; return; }
        if (piv != col) {
            for (int c = 0; c < 4; ++c) {
                const double t = f->lu[piv][c];
                f->lu[piv][c] = f->lu[col][c];
                f->lu[col][c] = t;
            }
            const int tp = f->perm[piv];
            f->perm[piv] = f->perm[col];
            f->perm[col] = tp;
        }
        for (int r = col + 1; r < 4; ++r) {
            const double m = f->lu[r][col] / f->lu[col][col];
            f->lu[r][col] = m;
            for (int c = col + 1; c < 4; ++c) f->lu[r][c] -= m * f->lu[col][c];
        }
    }
}

static void lu_solve(const lu4* f, const double b[4], double x[4]) {
    double y[4];
    for (int i = 0; i < 4; ++i) {
        double s = b[f->perm[i]];
        for (int j = 0; j < i; ++j) s -= f->lu[i][j] * y[j];
        y[i] = s;
    }
    for (int i = 3; i >= 0; --i) {
        double s = y[i];
        for (int j = i + 1; j < 4; ++j) s -= f->lu[i][j] * x[j];
        x[i] = s / f->lu[i][i];
    }
}

/* ------------------------------------------------------------------------ */
/* COO -> CSR, sparse.cpp:12-44: stable order by (row, col), duplicates
 * summed in insertion order.                                               */

static int triplets_to_csr(int64_t rows, int64_t nnz_in, const int64_t* tr, const int32_t* tc,
                           const double* tv, int64_t* rowptr, int32_t* col, double* val,
                           int64_t* nnz_out) {
    int64_t* cnt = (int64_t*)calloc((size_t)rows + 2, sizeof(int64_t));
    int64_t* order = (int64_t*)malloc((size_t)(nnz_in + 1) * sizeof(int64_t));
    if (!cnt || !order) { free(cnt); free(order); return fail(2, "out of memory"); }
    for (int64_t i = 0; i < nnz_in; ++i) cnt[tr[i] + 1]++;
    for (int64_t r = 0; r < rows; ++r) cnt[r + 1] += cnt[r];
    for (int64_t i = 0; i < nnz_in; ++i) order[cnt[tr[i]]++] = i; /* stable by row */
    /* cnt[r] now = end of row r; rows start at end of r-1 */
    int64_t out = 0, start = 0;
    rowptr[0] = 0;
    for (int64_t r = 0; r < rows; ++r) {
        const int64_t end = cnt[r];
        /* stable insertion sort of order[start..end) by column */
        for (int64_t i = start + 1; i < end; ++i) {
            const int64_t v = order[i];
            int64_t j = i - 1;
            while (j >= start && tc[order[j]] > tc[v]) {
                order[j + 1] = order[j];
                --j;
            }
            order[j + 1] = v;
        }
        int32_t prev = -1;
        const int64_t row_begin = out;
        for (int64_t i = start; i < end; ++i) {
            const int64_t idx = order[i];
            if (out > row_begin && tc[idx] == prev) {
                val[out - 1] += tv[idx];
            } else {
                col[out] = tc[idx];
                val[out] = tv[idx];
                prev = tc[idx];
                ++out;
            }
        }
        rowptr[r + 1] = out;
        start = end;
    }
    *nnz_out = out;
    free(cnt);
    free(order);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* assemble_system (assembly.cpp:106-138) + build_schur (solver.cpp:90-147) */

int or_assemble_condense(int64_t nc, int64_t ne, const double* coords, const int32_t* tets,
                         int64_t nf, const int32_t* faces, const int32_t* face_of_slot,
                         const int8_t* sigma, const int64_t* face_slots,
                         const uint8_t* face_class, const int32_t* mrow, const double* area,
                         int64_t l, const or_problem* prob, double* a_blocks, double* slot_coef_out,
                         int32_t* slot_mrow_out, double* rhs_out, double* bd_out,
                         int64_t* c_rowptr, int32_t* c_col, double* c_val, int64_t* s_rowptr,
                         int32_t* s_col, double* s_val, double* rhs_neg, int64_t* s_nnz) {
    (void)nc;
    const int kind = prob ? prob->kind : 0;
    const double cc = prob ? prob->c : 1.0;
    int rc = 0;
    double* A = (double*)malloc((size_t)(16 * ne + 1) * sizeof(double));
    double* coef = (double*)malloc((size_t)(4 * ne + 1) * sizeof(double));
    int32_t* row = (int32_t*)malloc((size_t)(4 * ne + 1) * sizeof(int32_t));
    double* b = (double*)calloc((size_t)(4 * ne + 1), sizeof(double));
    double* bd = (double*)calloc((size_t)(l + 1), sizeof(double));
    if (!A || !coef || !row || !b || !bd) { rc = fail(2, "out of memory"); goto done; }

    /* element blocks and C(T) entries (assembly.cpp:115-130) */
    for (int64_t t = 0; t < ne && !rc; ++t) {
        double Ac[3];
        coef_of(prob, t, Ac);
        local_mats lm;
        rc = local_stiffness_mass(coords, tets + 4 * t, t, Ac, cc, &lm);
        if (rc) break;
        memcpy(A + 16 * t, lm.a, sizeof lm.a);
        for (int k = 0; k < 4; ++k) {
            const int64_t slot = 4 * t + k;
            const int32_t f = face_of_slot[slot];
            row[slot] = mrow[f];
            coef[slot] = (double)sigma[slot] * area[f] / 3.0;
        }
    }
    if (rc) goto done;

    /* load vector, Gauss branch (assembly.cpp:64-78) */
    {
        double lam[4 * 64], w[64];
        or_tet_rule(5, lam, w);
        for (int64_t t = 0; t < ne; ++t) {
            const int32_t* e = tets + 4 * t;
            const v3 p[4] = {node(coords, e[0]), node(coords, e[1]), node(coords, e[2]), node(coords, e[3])};
            const double vol = fabs(vdot(vcross(vsub(p[1], p[0]), vsub(p[2], p[0])), vsub(p[3], p[0]))) / 6.0;
            double Ac[3];
            coef_of(prob, t, Ac);
            for (int q = 0; q < 64; ++q) {
                const double* L = lam + 4 * q;
                const v3 x = vadd(vadd(vadd(vmul(p[0], L[0]), vmul(p[1], L[1])), vmul(p[2], L[2])), vmul(p[3], L[3]));
                const double fw = vol * w[q] * orp_f(kind, x.x, x.y, x.z, Ac, cc);
                for (int v = 0; v < 4; ++v) b[4 * t + v] += fw * L[v];
            }
        }
    }
    /* neumann_vector (assembly.cpp:81-94) then rhs = b + LN (135) */
    {
        double* ln = (double*)calloc((size_t)(4 * ne + 1), sizeof(double));
        for (int64_t f = 0; f < nf && !rc; ++f) {
            if (face_class[f] != 2) continue;
            const int64_t slot = face_slots[2 * f];
            const int64_t t = slot / 4;
            const int k = (int)(slot % 4);
            double ar;
            v3 un;
            rc = face_geom(coords, faces + 3 * f, &ar, &un);
            if (rc) break;
            const v3 cen = face_centroid(coords, faces + 3 * f);
            double Ac[3];
            coef_of(prob, t, Ac);
            const double nn[3] = {un.x, un.y, un.z};
            const double gc = orp_g(kind, cen.x, cen.y, cen.z, nn, Ac);
            for (int v = 0; v < 3; ++v) ln[4 * t + kFaceVerts[k][v]] += ar * gc / 3.0;
        }
        for (int64_t i = 0; i < 4 * ne; ++i) b[i] += ln[i];
        free(ln);
        if (rc) goto done;
    }
    /* dirichlet_vector (assembly.cpp:96-104) */
    for (int64_t f = 0; f < nf; ++f) {
        if (face_class[f] != 1) continue;
        const v3 cen = face_centroid(coords, faces + 3 * f);
        bd[mrow[f]] = area[f] * orp_u(kind, cen.x, cen.y, cen.z);
    }

    if (a_blocks) memcpy(a_blocks, A, (size_t)(16 * ne) * sizeof(double));
    if (slot_coef_out) memcpy(slot_coef_out, coef, (size_t)(4 * ne) * sizeof(double));
    if (slot_mrow_out) memcpy(slot_mrow_out, row, (size_t)(4 * ne) * sizeof(int32_t));
    if (rhs_out) memcpy(rhs_out, b, (size_t)(4 * ne) * sizeof(double));
    if (bd_out) memcpy(bd_out, bd, (size_t)l * sizeof(double));

    /* C as CSR (assembly.cpp:121-130) */
    if (c_rowptr) {
        int64_t* tr = (int64_t*)malloc((size_t)(12 * ne + 1) * sizeof(int64_t));
        int32_t* tc = (int32_t*)malloc((size_t)(12 * ne + 1) * sizeof(int32_t));
        double* tv = (double*)malloc((size_t)(12 * ne + 1) * sizeof(double));
        int64_t n = 0, nnz;
        for (int64_t t = 0; t < ne; ++t)
            for (int k = 0; k < 4; ++k) {
                const int64_t slot = 4 * t + k;
                if (row[slot] < 0) continue;
                for (int v = 0; v < 3; ++v) {
                    tr[n] = row[slot];
                    tc[n] = (int32_t)(4 * t + kFaceVerts[k][v]);
                    tv[n++] = coef[slot];
                }
            }
        rc = triplets_to_csr(l, n, tr, tc, tv, c_rowptr, c_col, c_val, &nnz);
        free(tr);
        free(tc);
        free(tv);
        if (rc) goto done;
    }

    /* build_schur (solver.cpp:90-147) */
    if (s_rowptr) {
        int64_t* tr = (int64_t*)malloc((size_t)(16 * ne + 1) * sizeof(int64_t));
        int32_t* tc = (int32_t*)malloc((size_t)(16 * ne + 1) * sizeof(int32_t));
        double* tv = (double*)malloc((size_t)(16 * ne + 1) * sizeof(double));
        double* sl = (double*)malloc((size_t)(16 * ne + 1) * sizeof(double));
        double* rl = (double*)malloc((size_t)(4 * ne + 1) * sizeof(double));
        int64_t first_singular = -1;
        for (int64_t t = 0; t < ne; ++t) {
            lu4 lu;
            lu_factor((const double(*)[4])(A + 16 * t), &lu);
            if (lu.singular) {
                if (first_singular < 0) first_singular = t;
                continue;
            }
            double c[4][4] = {{0}};
            for (int r = 0; r < 4; ++r) { /* local_c_rows, solver.cpp:33-40 */
                if (row[4 * t + r] < 0) continue;
                for (int v = 0; v < 3; ++v) c[r][kFaceVerts[r][v]] = coef[4 * t + r];
            }
            double ainv_c[4][4], ainv_b[4];
            for (int r = 0; r < 4; ++r) lu_solve(&lu, c[r], ainv_c[r]);
            lu_solve(&lu, b + 4 * t, ainv_b);
            for (int r = 0; r < 4; ++r) {
                double rb = 0.0;
                for (int p = 0; p < 4; ++p) rb += c[r][p] * ainv_b[p];
                rl[4 * t + r] = rb;
                for (int q = 0; q < 4; ++q) {
                    double s = 0.0;
                    for (int p = 0; p < 4; ++p) s += c[r][p] * ainv_c[q][p];
                    sl[16 * t + 4 * r + q] = s;
                }
            }
        }
        if (first_singular >= 0) {
            rc = fail(2, "degenerate element block %lld", (long long)(first_singular + 1));
        } else {
            int64_t n = 0;
            memcpy(rhs_neg, bd, (size_t)l * sizeof(double));
            for (int64_t t = 0; t < ne; ++t)
                for (int r = 0; r < 4; ++r) {
                    const int32_t rr = row[4 * t + r];
                    if (rr < 0) continue;
                    rhs_neg[rr] -= rl[4 * t + r];
                    for (int q = 0; q < 4; ++q) {
                        const int32_t cq = row[4 * t + q];
                        if (cq < 0) continue;
                        tr[n] = rr;
                        tc[n] = cq;
                        tv[n++] = sl[16 * t + 4 * r + q];
                    }
                }
            rc = triplets_to_csr(l, n, tr, tc, tv, s_rowptr, s_col, s_val, s_nnz);
        }
        free(tr);
        free(tc);
        free(tv);
        free(sl);
        free(rl);
    }
done:
    free(A);
    free(coef);
    free(row);
    free(b);
    free(bd);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* pcg_jacobi, sparse.cpp:157-212                                            */

static double norm2(const double* v, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
    return sqrt(s);
}

static void csr_mul(int64_t n, const int64_t* rp, const int32_t* col, const double* val,
                    const double* x, double* y) {
    for (int64_t r = 0; r < n; ++r) {
        double s = 0.0;
        for (int64_t k = rp[r]; k < rp[r + 1]; ++k) s += val[k] * x[col[k]];
        y[r] = s;
    }
}

int or_pcg(int64_t n, const int64_t* rowptr, const int32_t* col, const double* val,
           const double* b, double* x, double tol, double abs_tol, int64_t max_iter,
           double res[3]) {
    for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
    const double bnorm = norm2(b, n);
    res[0] = 0.0;
    res[1] = 0.0;
    res[2] = 1.0;
    if (bnorm == 0.0) return 0;
    const int64_t mi = max_iter > 0 ? max_iter : 10 * n;
    const double stop = abs_tol > 0.0 ? fmin(tol * bnorm, abs_tol) : tol * bnorm;
    double* d = (double*)malloc((size_t)n * sizeof(double));
    double* r = (double*)malloc((size_t)n * sizeof(double));
    double* z = (double*)malloc((size_t)n * sizeof(double));
    double* p = (double*)malloc((size_t)n * sizeof(double));
    double* q = (double*)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) { /* CsrMatrix::diagonal, sparse.cpp:60-66 */
        double di = 0.0;
        for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k)
            if (col[k] == i) di += val[k];
        d[i] = di != 0.0 ? 1.0 / di : 1.0;
    }
    memcpy(r, b, (size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) z[i] = d[i] * r[i];
    memcpy(p, z, (size_t)n * sizeof(double));
    double rz = 0.0;
    for (int64_t i = 0; i < n; ++i) rz += r[i] * z[i];
    int rc = 0;
    res[2] = 0.0;
    res[1] = 1.0;
    for (int64_t it = 1; it <= mi; ++it) {
        csr_mul(n, rowptr, col, val, p, q);
        double pq = 0.0;
        for (int64_t i = 0; i < n; ++i) pq += p[i] * q[i];
        if (pq <= 0.0) { rc = fail(3, "pcg: operator is not positive definite"); break; }
        const double alpha = rz / pq;
        for (int64_t i = 0; i < n; ++i) {
            x[i] += alpha * p[i];
            r[i] -= alpha * q[i];
        }
        res[0] = (double)it;
        const double rnorm = norm2(r, n);
        res[1] = rnorm / bnorm;
        if (rnorm <= stop) { res[2] = 1.0; break; }
        double rz_new = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            z[i] = d[i] * r[i];
            rz_new += r[i] * z[i];
        }
        const double beta = rz_new / rz;
        rz = rz_new;
        for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
    free(d); free(r); free(z); free(p); free(q);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* solve_schur_parallel (solver.cpp:149-186) + verify_solution (44-76)       */

/* Componentwise magnitudes for per-entry parity of the load data (TEST
 * INFRASTRUCTURE; no reference counterpart).  The GPU and the reference
 * evaluate sin/cos/exp differently (libdevice / series vs glibc libm), so an
 * entry of B_T or rhs_neg that is a cancelling sum cannot agree to 1e-12 of
 * its own size; it agrees to 1e-12 of the magnitude its summands carry:
 *   rhs_scale[4t+v] = sum_q |V w_q f(x_q)| lambda_v + sum |Neumann terms|
 *                    (the summands of assembly.cpp:75 and :91),
 *   rhsneg_scale[R] = |b_D[R]| + sum_T sum_p |c_r[p]| (|A_T^-1| rhs_scale_T)_p
 *                    (first-order propagation of B_T through
 *                    r_T = C A^-1 B, solver.cpp:111-119, 133-138). */
int or_entry_scales(int64_t nc, int64_t ne, const double* coords, const int32_t* tets, int64_t nf,
                    const int32_t* faces, const int32_t* face_of_slot, const int8_t* sigma,
                    const int64_t* face_slots, const uint8_t* face_class, const int32_t* mrow,
                    const double* area, int64_t l, const or_problem* prob, double* rhs_scale,
                    double* rhsneg_scale) {
    (void)nc;
    const int kind = prob ? prob->kind : 0;
    const double cc = prob ? prob->c : 1.0;
    int rc = 0;
    double lam[4 * 64], w[64];
    or_tet_rule(5, lam, w);
    for (int64_t i = 0; i < 4 * ne; ++i) rhs_scale[i] = 0.0;
    for (int64_t t = 0; t < ne; ++t) {
        const int32_t* e = tets + 4 * t;
        const v3 p[4] = {node(coords, e[0]), node(coords, e[1]), node(coords, e[2]), node(coords, e[3])};
        const double vol = fabs(vdot(vcross(vsub(p[1], p[0]), vsub(p[2], p[0])), vsub(p[3], p[0]))) / 6.0;
        double Ac[3];
        coef_of(prob, t, Ac);
        for (int q = 0; q < 64; ++q) {
            const double* L = lam + 4 * q;
            const v3 x = vadd(vadd(vadd(vmul(p[0], L[0]), vmul(p[1], L[1])), vmul(p[2], L[2])), vmul(p[3], L[3]));
            const double fw = fabs(vol * w[q] * orp_f(kind, x.x, x.y, x.z, Ac, cc));
            for (int v = 0; v < 4; ++v) rhs_scale[4 * t + v] += fw * L[v];
        }
    }
    for (int64_t f = 0; f < nf && !rc; ++f) {
        if (face_class[f] != 2) continue;
        const int64_t slot = face_slots[2 * f];
        const int64_t t = slot / 4;
        const int k = (int)(slot % 4);
        double ar;
        v3 un;
        rc = face_geom(coords, faces + 3 * f, &ar, &un);
        if (rc) break;
        const v3 cen = face_centroid(coords, faces + 3 * f);
        double Ac[3];
        coef_of(prob, t, Ac);
        const double nn[3] = {un.x, un.y, un.z};
        const double gc = orp_g(kind, cen.x, cen.y, cen.z, nn, Ac);
        for (int v = 0; v < 3; ++v) rhs_scale[4 * t + kFaceVerts[k][v]] += fabs(ar * gc / 3.0);
    }
    if (rc) return rc;
    for (int64_t r = 0; r < l; ++r) rhsneg_scale[r] = 0.0;
    for (int64_t f = 0; f < nf; ++f) {
        if (face_class[f] != 1) continue;
        const v3 cen = face_centroid(coords, faces + 3 * f);
        rhsneg_scale[mrow[f]] = fabs(area[f] * orp_u(kind, cen.x, cen.y, cen.z));
    }
    for (int64_t t = 0; t < ne && !rc; ++t) {
        double Ac[3];
        coef_of(prob, t, Ac);
        local_mats lm;
        rc = local_stiffness_mass(coords, tets + 4 * t, t, Ac, cc, &lm);
        if (rc) break;
        lu4 lu;
        lu_factor(lm.a, &lu);
        if (lu.singular) continue;
        double ainv[4][4]; /* columns of A^-1 */
        for (int j = 0; j < 4; ++j) {
            double ej[4] = {0.0, 0.0, 0.0, 0.0};
            ej[j] = 1.0;
            lu_solve(&lu, ej, ainv[j]);
        }
        double prop[4];
        for (int pp = 0; pp < 4; ++pp) {
            prop[pp] = 0.0;
            for (int j = 0; j < 4; ++j) prop[pp] += fabs(ainv[j][pp]) * rhs_scale[4 * t + j];
        }
        for (int r = 0; r < 4; ++r) {
            const int64_t slot = 4 * t + r;
            const int32_t R = mrow[face_of_slot[slot]];
            if (R < 0) continue;
            const double cf = fabs((double)sigma[slot] * area[face_of_slot[slot]] / 3.0);
            double s = 0.0;
            for (int v = 0; v < 3; ++v) s += cf * prop[kFaceVerts[r][v]];
            rhsneg_scale[R] += s;
        }
    }
    return rc;
}

int or_solve_schur(int64_t nc, int64_t ne, const double* coords, const int32_t* tets,
                   const or_problem* prob, int64_t l, const double* slot_coef,
                   const int32_t* slot_mrow, const double* rhs, const double* bd,
                   const int64_t* c_rowptr, const int32_t* c_col, const double* c_val,
                   const int64_t* s_rowptr, const int32_t* s_col, const double* s_val,
                   const double* rhs_neg, double tol, int64_t max_iter, double* u,
                   double* lambda, double stats[3]) {
    (void)nc;
    const double cc = prob ? prob->c : 1.0;
    const int64_t n = 4 * ne;
    /* inner_cg_options, solver.cpp:78-86 */
    const double abs_tol = 0.2 * tol * hypot(norm2(rhs, n), norm2(bd, l));
    const int64_t mi = max_iter > 0 ? max_iter : 10 * (l > 1 ? l : 1);
    double res[3];
    int rc = or_pcg(l, s_rowptr, s_col, s_val, rhs_neg, lambda, tol, abs_tol, mi, res);
    stats[0] = res[0];
    if (rc) return rc;
    if (res[2] == 0.0) {
        return fail(3, "schur: conjugate gradients stalled at relative residual %f after %lld iterations",
                    res[1], (long long)res[0]);
    }
    /* recovery (solver.cpp:168-181) */
    double* r1 = (double*)malloc((size_t)(n + 1) * sizeof(double));
    for (int64_t t = 0; t < ne && !rc; ++t) {
        double Ac[3];
        coef_of(prob, t, Ac);
        local_mats lm;
        rc = local_stiffness_mass(coords, tets + 4 * t, t, Ac, cc, &lm);
        if (rc) break;
        lu4 lu;
        lu_factor(lm.a, &lu);
        double rr[4] = {rhs[4 * t], rhs[4 * t + 1], rhs[4 * t + 2], rhs[4 * t + 3]};
        for (int r = 0; r < 4; ++r) {
            const int32_t row = slot_mrow[4 * t + r];
            if (row < 0) continue;
            for (int v = 0; v < 3; ++v) rr[kFaceVerts[r][v]] += slot_coef[4 * t + r] * lambda[row];
        }
        lu_solve(&lu, rr, u + 4 * t);
        /* verify: A U - rhs (solver.cpp:45-50) */
        for (int i = 0; i < 4; ++i) {
            double s = 0.0;
            for (int j = 0; j < 4; ++j) s += lm.a[i][j] * u[4 * t + j];
            r1[4 * t + i] = s - rhs[4 * t + i];
        }
    }
    if (rc) { free(r1); return rc; }
    /* - C' Lambda (solver.cpp:51-53, multiply_transpose sparse.cpp:54-58) */
    double* ctl = (double*)calloc((size_t)(n + 1), sizeof(double));
    for (int64_t r = 0; r < l; ++r)
        for (int64_t k = c_rowptr[r]; k < c_rowptr[r + 1]; ++k) ctl[c_col[k]] += c_val[k] * lambda[r];
    for (int64_t i = 0; i < n; ++i) r1[i] -= ctl[i];
    /* C U - b_D (solver.cpp:55-62) */
    double* r2 = (double*)malloc((size_t)(l + 1) * sizeof(double));
    csr_mul(l, c_rowptr, c_col, c_val, u, r2);
    double bd_inf = 0.0, r2_inf = 0.0;
    for (int64_t i = 0; i < l; ++i) {
        bd_inf = fmax(bd_inf, fabs(bd[i]));
        r2[i] -= bd[i];
        r2_inf = fmax(r2_inf, fabs(r2[i]));
    }
    const double rhs_norm = hypot(norm2(rhs, n), norm2(bd, l));
    const double res_norm = hypot(norm2(r1, n), norm2(r2, l));
    stats[1] = rhs_norm > 0.0 ? res_norm / rhs_norm : res_norm;
    stats[2] = r2_inf / (1.0 + bd_inf);
    const double nr = norm2(rhs, n);
    const int ok = stats[1] <= tol && norm2(r1, n) <= tol * fmax(nr, 1e-300) &&
                   norm2(r2, l) <= tol * (1.0 + norm2(bd, l));
    free(r1);
    free(ctl);
    free(r2);
    if (!ok) return fail(3, "solver 'schur' missed the residual target: %g > %g", stats[1], tol);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Streaming connectivity digests (TEST INFRASTRUCTURE).  Config 2's level 7
 * (215M tets) does not fit the full oracle tables in host memory (the E2T
 * alone is 41 GB, SURVEY.md 8(c) "Limits"), so its connectivity is checked
 * through SHA-256 digests of the arrays the reference defines, computed here
 * in one element-order pass with the same first-occurrence rules:
 *   edges: num_edges (connectivity.cpp:22-37), ids in first-occurrence order;
 *   faces: a face is first seen at its owner slot (the lower element, the
 *          slot faces_up emits, connectivity.cpp:72-86), whose oriented
 *          tuple is stored; face ids in that order; the second slot gets
 *          sigma from same_cycle (connectivity.cpp:104-108, 145);
 *          face_area from face_area_and_normal (mesh.cpp:76-84);
 *          class 1 (Dirichlet) for faces with one slot (config 2 lists every
 *          boundary face as Dirichlet), multiplier row = face id.
 * SHA-256 is FIPS 180-4, restated here. */

typedef struct {
    uint32_t h[8];
    uint64_t len;
    uint8_t buf[64];
    int nbuf;
} sha256;

static const uint32_t kSha[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

static void sha_init(sha256* s) {
    static const uint32_t h0[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                                   0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    memcpy(s->h, h0, sizeof h0);
    s->len = 0;
    s->nbuf = 0;
}

static void sha_block(sha256* s, const uint8_t* p) {
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
        w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
        const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
        const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
        w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = s->h[0], b = s->h[1], c = s->h[2], d = s->h[3], e = s->h[4], f = s->h[5], g = s->h[6],
             h = s->h[7];
    for (int i = 0; i < 64; ++i) {
        const uint32_t t1 = h + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + kSha[i] + w[i];
        const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
        h = g;
        g = f;
        f = e;
        e = d + t1;
        d = c;
        c = b;
        b = a;
        a = t1 + t2;
    }
    s->h[0] += a; s->h[1] += b; s->h[2] += c; s->h[3] += d;
    s->h[4] += e; s->h[5] += f; s->h[6] += g; s->h[7] += h;
}

static void sha_update(sha256* s, const void* data, size_t n) {
    const uint8_t* p = (const uint8_t*)data;
    s->len += n;
    while (n) {
        if (s->nbuf == 0 && n >= 64) {
            sha_block(s, p);
            p += 64;
            n -= 64;
            continue;
        }
        const size_t k = (size_t)(64 - s->nbuf) < n ? (size_t)(64 - s->nbuf) : n;
        memcpy(s->buf + s->nbuf, p, k);
        s->nbuf += (int)k;
        p += k;
        n -= k;
        if (s->nbuf == 64) {
            sha_block(s, s->buf);
            s->nbuf = 0;
        }
    }
}

static void sha_final(sha256* s, uint8_t out[32]) {
    const uint64_t bits = s->len * 8;
    const uint8_t one = 0x80, zero = 0;
    sha_update(s, &one, 1);
    while (s->nbuf != 56) sha_update(s, &zero, 1);
    uint8_t lb[8];
    for (int i = 0; i < 8; ++i) lb[i] = (uint8_t)(bits >> (56 - 8 * i));
    sha_update(s, lb, 8);
    for (int i = 0; i < 8; ++i) {
        out[4 * i] = (uint8_t)(s->h[i] >> 24);
        out[4 * i + 1] = (uint8_t)(s->h[i] >> 16);
        out[4 * i + 2] = (uint8_t)(s->h[i] >> 8);
        out[4 * i + 3] = (uint8_t)s->h[i];
    }
}

void or_sha256(const void* data, int64_t n, uint8_t out[32]) {
    sha256 s;
    sha_init(&s);
    sha_update(&s, data, (size_t)n);
    sha_final(&s, out);
}

static int same_cycle3(const int32_t a[3], const int32_t b[3]) {
    return (a[0] == b[0] && a[1] == b[1] && a[2] == b[2]) || (a[0] == b[1] && a[1] == b[2] && a[2] == b[0]) ||
           (a[0] == b[2] && a[1] == b[0] && a[2] == b[1]);
}

int or_conn_digests(int64_t nc, int64_t ne, const int32_t* tets, const double* coords, uint8_t* digests,
                    int64_t counts[2]) {
    enum { D_EN, D_EOS, D_F, D_FOS, D_SIG, D_FS, D_AREA, D_CLS, D_MROW, ND };
    sha256 sh[ND];
    for (int i = 0; i < ND; ++i) sha_init(&sh[i]);
    edge_table et;
    et.nc = nc;
    hmap fm;
    if (hmap_init(&et.map, 2 * ne + 8) || hmap_init(&fm, 2 * ne + 8)) return fail(2, "out of memory");
    /* per face: owner slot, second slot (filled later), the stored tuple
     * for the sigma test of the second slot */
    int64_t cap = 2 * ne + ne / 16 + 1024; /* nF ~ 2 nE + boundary / 2; grown on demand */
    int32_t* owner = (int32_t*)malloc((size_t)cap * sizeof(int32_t));
    int32_t* mate = (int32_t*)malloc((size_t)cap * sizeof(int32_t));
    if (!owner || !mate) return fail(2, "out of memory");
    int64_t ned = 0, nf = 0;
    for (int64_t t = 0; t < ne; ++t) {
        const int32_t* e = tets + 4 * t;
        int32_t eos[6];
        for (int k = 0; k < 6; ++k) {
            int32_t a = e[kEdgeVerts[k][0]], b = e[kEdgeVerts[k][1]];
            if (a > b) { const int32_t x = a; a = b; b = x; }
            int ins;
            eos[k] = hmap_try_emplace(&et.map, (uint64_t)a * (uint64_t)nc + (uint64_t)b, (int32_t)ned, &ins);
            if (ins) {
                const int32_t pr[2] = {a, b};
                sha_update(&sh[D_EN], pr, sizeof pr);
                ++ned;
            }
        }
        sha_update(&sh[D_EOS], eos, sizeof eos);
        int32_t fos[4];
        int8_t sig[4];
        for (int k = 0; k < 4; ++k) {
            int32_t f[3];
            oriented_face(e, k, f);
            int32_t v[3] = {f[0], f[1], f[2]};
            /* sorted node set -> (edge of the two smallest, largest) */
            if (v[0] > v[1]) { const int32_t x = v[0]; v[0] = v[1]; v[1] = x; }
            if (v[1] > v[2]) { const int32_t x = v[1]; v[1] = v[2]; v[2] = x; }
            if (v[0] > v[1]) { const int32_t x = v[0]; v[0] = v[1]; v[1] = x; }
            const int32_t e01 = pair_to_edge(&et, v[0], v[1]);
            int ins;
            const int32_t id = hmap_try_emplace(&fm, (uint64_t)e01 * (uint64_t)nc + (uint64_t)v[2], (int32_t)nf, &ins);
            fos[k] = id;
            if (ins) {
                if (nf == cap) {
                    cap *= 2;
                    owner = (int32_t*)realloc(owner, (size_t)cap * sizeof(int32_t));
                    mate = (int32_t*)realloc(mate, (size_t)cap * sizeof(int32_t));
                    if (!owner || !mate) return fail(2, "out of memory");
                }
                owner[nf] = (int32_t)(4 * t + k);
                mate[nf] = -1;
                sha_update(&sh[D_F], f, sizeof f);
                double ar;
                v3 un;
                if (face_geom(coords, f, &ar, &un)) ar = 0.0;
                sha_update(&sh[D_AREA], &ar, sizeof ar);
                sig[k] = 1;
                ++nf;
            } else {
                mate[id] = (int32_t)(4 * t + k);
                const int64_t os = owner[id];
                int32_t g[3];
                oriented_face(tets + 4 * (os / 4), (int)(os % 4), g);
                sig[k] = same_cycle3(f, g) ? 1 : -1;
            }
        }
        sha_update(&sh[D_FOS], fos, sizeof fos);
        sha_update(&sh[D_SIG], sig, sizeof sig);
    }
    for (int64_t f = 0; f < nf; ++f) {
        const int64_t fs[2] = {owner[f], mate[f]};
        sha_update(&sh[D_FS], fs, sizeof fs);
        const uint8_t cls = mate[f] < 0 ? 1 : 0;
        sha_update(&sh[D_CLS], &cls, 1);
        const int32_t row = (int32_t)f;
        sha_update(&sh[D_MROW], &row, sizeof row);
    }
    for (int i = 0; i < ND; ++i) sha_final(&sh[i], digests + 32 * i);
    counts[0] = ned;
    counts[1] = nf;
    free(owner);
    free(mate);
    hmap_free(&et.map);
    hmap_free(&fm);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* error norms, analysis.cpp:51-105 (+ L2 extension)                        */

double or_mesh_diameter(int64_t nc, int64_t ne, const double* coords, const int32_t* tets) {
    (void)nc;
    double h = 0.0;
    for (int64_t t = 0; t < ne; ++t) {
        double d2 = 0.0;
        for (int i = 0; i < 4; ++i)
            for (int j = i + 1; j < 4; ++j) {
                const v3 d = vsub(node(coords, tets[4 * t + i]), node(coords, tets[4 * t + j]));
                d2 = fmax(d2, vdot(d, d));
            }
        h = fmax(h, sqrt(d2));
    }
    return h;
}

int or_errors(int64_t nc, int64_t ne, const double* coords, const int32_t* tets,
              const int32_t* face_of_slot, const int8_t* sigma, const int32_t* mrow,
              const or_problem* prob, const double* u, const double* lambda, double out[3]) {
    const int kind = prob ? prob->kind : 0;
    const double cc = prob ? prob->c : 1.0;
    double lam[4 * 216], w[216];
    or_tet_rule(9, lam, w);
    const double h = or_mesh_diameter(nc, ne, coords, tets);
    const double inv_h2 = 1.0 / (h * h);
    double acc_y = 0.0, acc_l2 = 0.0, acc_k = 0.0;
    for (int64_t t = 0; t < ne; ++t) {
        const int32_t* e = tets + 4 * t;
        const v3 p[4] = {node(coords, e[0]), node(coords, e[1]), node(coords, e[2]), node(coords, e[3])};
        double Ac[3];
        coef_of(prob, t, Ac);
        local_mats lm;
        int rc = local_stiffness_mass(coords, e, t, Ac, cc, &lm);
        if (rc) return rc;
        v3 guh = {0.0, 0.0, 0.0};
        for (int v = 0; v < 4; ++v) guh = vadd(guh, vmul(lm.g[v], u[4 * t + v]));
        for (int q = 0; q < 216; ++q) {
            const double* L = lam + 4 * q;
            const v3 x = vadd(vadd(vadd(vmul(p[0], L[0]), vmul(p[1], L[1])), vmul(p[2], L[2])), vmul(p[3], L[3]));
            double uh = 0.0;
            for (int v = 0; v < 4; ++v) uh += L[v] * u[4 * t + v];
            double g[3];
            orp_grad(kind, x.x, x.y, x.z, g);
            const v3 dg = {g[0] - guh.x, g[1] - guh.y, g[2] - guh.z};
            const double dv = orp_u(kind, x.x, x.y, x.z) - uh;
            acc_y += lm.volume * w[q] * (vdot(dg, dg) + inv_h2 * dv * dv);
            const double vol = fabs(vdot(vcross(vsub(p[1], p[0]), vsub(p[2], p[0])), vsub(p[3], p[0]))) / 6.0;
            acc_l2 += vol * w[q] * (dv * dv);
        }
        /* multiplier_norm_error, analysis.cpp:78-105 */
        static const double tl[3][3] = {{0.5, 0.5, 0.0}, {0.0, 0.5, 0.5}, {0.5, 0.0, 0.5}};
        for (int k = 0; k < 4; ++k) {
            const int64_t slot = 4 * t + k;
            const int32_t f = face_of_slot[slot];
            if (mrow[f] < 0) continue;
            int32_t tri[3];
            oriented_face(e, k, tri);
            double ar;
            v3 un;
            rc = face_geom(coords, tri, &ar, &un);
            if (rc) return rc;
            const double kappa_h = (double)sigma[slot] * lambda[mrow[f]];
            const v3 q0 = node(coords, tri[0]), q1 = node(coords, tri[1]), q2 = node(coords, tri[2]);
            for (int qq = 0; qq < 3; ++qq) {
                const v3 x = vadd(vadd(vmul(q0, tl[qq][0]), vmul(q1, tl[qq][1])), vmul(q2, tl[qq][2]));
                const double nn[3] = {un.x, un.y, un.z};
                const double diff = orp_g(kind, x.x, x.y, x.z, nn, Ac) - kappa_h;
                acc_k += h * ar * (1.0 / 3.0) * diff * diff;
            }
        }
    }
    out[0] = sqrt(acc_y);
    out[1] = sqrt(acc_k);
    out[2] = sqrt(acc_l2);
    return 0;
}
