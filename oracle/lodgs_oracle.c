/* lodgs_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU checker, never the product.
 *
 * Plain-C restatement of the reference per-frame render path.  Single
 * threaded; every worker-count in the reference is a pure timing knob
 * (worker_pool.hpp:13-18), so the restatement drops it.  See lodgs_oracle.h.
 * Compiled with -ffp-contract=off: every a*b+c below rounds twice, exactly as
 * the reference's scalar kernels (mark_core.hpp:12-15).
 */
#include "lodgs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* std::max / std::min semantics (NaN in the first argument propagates). */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }

/* ------------------------------------------------------------------ rng -- */
/* rng.hpp:11-33: std::mt19937_64 (published MT19937-64 parameters). */
#define MT_N 312
#define MT_M 156
void orc_rng_seed(orc_rng *r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
}

static void mt_twist(orc_rng *r) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < MT_N; ++i) {
        const uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->idx = 0;
}

uint64_t orc_rng_next_u64(orc_rng *r) {
    if (r->idx >= MT_N) mt_twist(r);
    uint64_t x = r->mt[r->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* rng.hpp:19 */
double orc_rng_next_double(orc_rng *r) {
    return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53;
}
/* rng.hpp:21 */
double orc_rng_uniform(orc_rng *r, double lo, double hi) {
    return lo + (hi - lo) * orc_rng_next_double(r);
}
/* rng.hpp:24 */
uint64_t orc_rng_next_below(orc_rng *r, uint64_t n) { return orc_rng_next_u64(r) % n; }
/* rng.hpp:28-33 */
uint64_t orc_mix_seed(uint64_t seed, uint64_t item) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ULL * (item + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
size_t orc_rng_sizeof(void) { return sizeof(orc_rng); }

/* ------------------------------------------------------- camera fixtures -- */
/* test_util.hpp:19-28 */
void orc_front_camera(uint32_t w, uint32_t h, double focal, orc_camera *c) {
    memset(c, 0, sizeof *c);
    c->width = w;
    c->height = h;
    c->fx = c->fy = focal;
    c->cx = w / 2.0;
    c->cy = h / 2.0;
    c->rotation[0] = c->rotation[4] = c->rotation[8] = 1.0;
    c->znear = 0.01;
    c->zfar = 1000.0;
}

static double dot3(const double a[3], const double b[3]) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

/* test_util.hpp:32-60 */
void orc_orbit_camera(orc_rng *r, uint32_t w, uint32_t h, double dist, orc_camera *c) {
    const double az = orc_rng_uniform(r, 0.0, 2.0 * 3.14159265358979);
    const double el = orc_rng_uniform(r, -0.9, 0.9);
    const double eye[3] = {dist * cos(el) * cos(az), dist * sin(el), dist * cos(el) * sin(az)};
    double zc[3] = {eye[0] * -1.0, eye[1] * -1.0, eye[2] * -1.0};
    const double zn = sqrt(dot3(zc, zc));
    for (int i = 0; i < 3; ++i) zc[i] = zc[i] * (1.0 / zn);
    double up[3] = {0, 1, 0};
    if (fabs(dot3(up, zc)) > 0.99) {
        up[0] = 1;
        up[1] = 0;
        up[2] = 0;
    }
    double xc[3] = {up[1] * zc[2] - up[2] * zc[1], up[2] * zc[0] - up[0] * zc[2],
                    up[0] * zc[1] - up[1] * zc[0]};
    const double xn = sqrt(dot3(xc, xc));
    for (int i = 0; i < 3; ++i) xc[i] = xc[i] * (1.0 / xn);
    const double yc[3] = {zc[1] * xc[2] - zc[2] * xc[1], zc[2] * xc[0] - zc[0] * xc[2],
                          zc[0] * xc[1] - zc[1] * xc[0]};
    orc_front_camera(w, h, orc_rng_uniform(r, 80.0, 260.0), c);
    for (int i = 0; i < 3; ++i) {
        c->rotation[i] = xc[i];
        c->rotation[3 + i] = yc[i];
        c->rotation[6 + i] = zc[i];
    }
    c->translation[0] = -(xc[0] * eye[0] + xc[1] * eye[1] + xc[2] * eye[2]);
    c->translation[1] = -(yc[0] * eye[0] + yc[1] * eye[1] + yc[2] * eye[2]);
    c->translation[2] = -(zc[0] * eye[0] + zc[1] * eye[1] + zc[2] * eye[2]);
}

/* ------------------------------------------------------------- geometry -- */
static void side_plane(double n0, double n1, double n2, double *p) {
    const double len = sqrt(n0 * n0 + n1 * n1 + n2 * n2);
    p[0] = n0 / len;
    p[1] = n1 / len;
    p[2] = n2 / len;
    p[3] = 0.0;
}

/* projection.cpp:11-38 */
void orc_camera_geom(const orc_camera *c, orc_geom *g) {
    memset(g, 0, sizeof *g);
    for (int i = 0; i < 9; ++i) g->rot[i] = c->rotation[i];
    for (int i = 0; i < 3; ++i) g->trans[i] = c->translation[i];
    g->fx = c->fx;
    g->fy = c->fy;
    g->cx = c->cx;
    g->cy = c->cy;
    g->width = c->width;
    g->height = c->height;
    g->znear = c->znear;
    g->zfar = c->zfar;
    g->planes[0][2] = 1;
    g->planes[0][3] = -g->znear;
    g->planes[1][2] = -1;
    g->planes[1][3] = g->zfar;
    side_plane(g->fx, 0, g->cx, g->planes[2]);
    side_plane(-g->fx, 0, g->width - g->cx, g->planes[3]);
    side_plane(0, g->fy, g->cy, g->planes[4]);
    side_plane(0, -g->fy, g->height - g->cy, g->planes[5]);
}

/* mark_core.hpp:24-116, operation for operation. */
void orc_mark_core(const orc_geom *g, float mx, float my, float mz, float sx, float sy, float sz,
                   float qw, float qx, float qy, float qz, double tau_r, orc_mark_out *o) {
    const double x = mx, y = my, z = mz;
    o->tx = (g->rot[0] * x + g->rot[1] * y) + (g->rot[2] * z + g->trans[0]);
    o->ty = (g->rot[3] * x + g->rot[4] * y) + (g->rot[5] * z + g->trans[1]);
    o->tz = (g->rot[6] * x + g->rot[7] * y) + (g->rot[8] * z + g->trans[2]);

    const double sm = smax(smax((double)sx, (double)sy), (double)sz);
    const double r3 = 3.0 * sm;
    int vis = 1;
    for (int p = 0; p < 6; ++p) {
        const double dist = (g->planes[p][0] * o->tx + g->planes[p][1] * o->ty) +
                            (g->planes[p][2] * o->tz + g->planes[p][3]);
        vis = vis && dist >= -r3;
    }
    o->vis = vis;
    o->z_ok = o->tz >= g->znear;

    const double w = qw, xq = qx, yq = qy, zq = qz;
    const double qn = sqrt(((w * w + xq * xq) + (yq * yq + zq * zq)));
    const double iw = w / qn, ix = xq / qn, iy = yq / qn, iz = zq / qn;
    const double m00 = 1.0 - 2.0 * (iy * iy + iz * iz);
    const double m01 = 2.0 * (ix * iy - iw * iz);
    const double m02 = 2.0 * (ix * iz + iw * iy);
    const double m10 = 2.0 * (ix * iy + iw * iz);
    const double m11 = 1.0 - 2.0 * (ix * ix + iz * iz);
    const double m12 = 2.0 * (iy * iz - iw * ix);
    const double m20 = 2.0 * (ix * iz - iw * iy);
    const double m21 = 2.0 * (iy * iz + iw * ix);
    const double m22 = 1.0 - 2.0 * (ix * ix + iy * iy);

    const double dsx = sx, dsy = sy, dsz = sz;
    const double v00 = m00 * dsx, v01 = m01 * dsy, v02 = m02 * dsz;
    const double v10 = m10 * dsx, v11 = m11 * dsy, v12 = m12 * dsz;
    const double v20 = m20 * dsx, v21 = m21 * dsy, v22 = m22 * dsz;
    const double s00 = (v00 * v00 + v01 * v01) + v02 * v02;
    const double s01 = (v00 * v10 + v01 * v11) + v02 * v12;
    const double s02 = (v00 * v20 + v01 * v21) + v02 * v22;
    const double s11 = (v10 * v10 + v11 * v11) + v12 * v12;
    const double s12 = (v10 * v20 + v11 * v21) + v12 * v22;
    const double s22 = (v20 * v20 + v21 * v21) + v22 * v22;

    const double *r = g->rot;
    const double b00 = (r[0] * s00 + r[1] * s01) + r[2] * s02;
    const double b01 = (r[0] * s01 + r[1] * s11) + r[2] * s12;
    const double b02 = (r[0] * s02 + r[1] * s12) + r[2] * s22;
    const double b10 = (r[3] * s00 + r[4] * s01) + r[5] * s02;
    const double b11 = (r[3] * s01 + r[4] * s11) + r[5] * s12;
    const double b12 = (r[3] * s02 + r[4] * s12) + r[5] * s22;
    const double b20 = (r[6] * s00 + r[7] * s01) + r[8] * s02;
    const double b21 = (r[6] * s01 + r[7] * s11) + r[8] * s12;
    const double b22 = (r[6] * s02 + r[7] * s12) + r[8] * s22;
    const double c00 = (b00 * r[0] + b01 * r[1]) + b02 * r[2];
    const double c01 = (b00 * r[3] + b01 * r[4]) + b02 * r[5];
    const double c02 = (b00 * r[6] + b01 * r[7]) + b02 * r[8];
    const double c11 = (b10 * r[3] + b11 * r[4]) + b12 * r[5];
    const double c12 = (b10 * r[6] + b11 * r[7]) + b12 * r[8];
    const double c22 = (b20 * r[6] + b21 * r[7]) + b22 * r[8];
    (void)b21;
    (void)b22;

    const double zc = smax(o->tz, 1e-12);
    const double inv_z = 1.0 / zc;
    const double inv_z2 = inv_z * inv_z;
    const double j00 = g->fx * inv_z;
    const double j02 = (0.0 - g->fx * o->tx) * inv_z2;
    const double j11 = g->fy * inv_z;
    const double j12 = (0.0 - g->fy * o->ty) * inv_z2;

    const double t00 = j00 * c00 + j02 * c02;
    const double t01 = j00 * c01 + j02 * c12;
    const double t02 = j00 * c02 + j02 * c22;
    const double t11 = j11 * c11 + j12 * c12;
    const double t12 = j11 * c12 + j12 * c22;
    o->a = (t00 * j00 + t02 * j02) + 0.3;
    o->b = t01 * j11 + t02 * j12;
    o->c = (t11 * j11 + t12 * j12) + 0.3;

    const double det = o->a * o->c - o->b * o->b;
    const double mid = 0.5 * (o->a + o->c);
    const double disc = sqrt(smax(mid * mid - det, 0.0));
    o->lambda_max = mid + disc;
    o->lambda_min = mid - disc;
    o->radius = 3.0 * sqrt(o->lambda_max);
    o->qpass = o->vis && o->z_ok && o->radius <= tau_r;
}

static void mark_node(const orc_geom *g, const orc_tree *t, uint64_t i, double tau_r,
                      orc_mark_out *o) {
    orc_mark_core(g, t->mean_x[i], t->mean_y[i], t->mean_z[i], t->scale_x[i], t->scale_y[i],
                  t->scale_z[i], t->quat_w[i], t->quat_x[i], t->quat_y[i], t->quat_z[i], tau_r,
                  o);
}

/* mark_scalar.cpp:7-19 */
void orc_mark(const orc_geom *g, const orc_tree *t, uint64_t begin, uint64_t end, double tau_r,
              uint8_t *vis, uint8_t *qpass, double *radius_out) {
    orc_mark_out o;
    for (uint64_t i = begin; i < end; ++i) {
        mark_node(g, t, i, tau_r, &o);
        vis[i] = o.vis ? 1 : 0;
        qpass[i] = o.qpass ? 1 : 0;
        if (radius_out) radius_out[i] = o.radius;
    }
}

/* --------------------------------------------------------------- filter -- */
/* filter.cpp:20-25 */
static int ancestor_disqualifies(const orc_tree *t, uint32_t n, const uint8_t *qpass) {
    for (uint32_t a = t->parent[n]; a != ORC_ROOT_PARENT; a = t->parent[a])
        if (qpass[a] && !t->leaf[a]) return 1;
    return 0;
}

static uint32_t level_end(const orc_tree *t, uint32_t l) {
    return l + 1 < t->n_levels ? t->level_offsets[l + 1] : (uint32_t)t->n;
}

/* filter.cpp:29-150. mode: oracle (:29-58), serial (:60-113), parallel (:115-150).
 * The parallel two-pass form and the literal oracle produce the same list by
 * construction; serial is the level-wise descent with its own visiting order. */
int orc_filter(const orc_tree *t, const orc_camera *cam, double tau_r, int mode,
               uint32_t *selected, uint64_t *n_selected, int32_t *passes, int32_t *barriers) {
    if (!(tau_r > 0)) return ORC_EVALIDATION; /* filter.cpp:14-18 */
    orc_geom g;
    orc_camera_geom(cam, &g);
    const uint64_t n = t->n;
    uint64_t ns = 0;
    if (mode != ORC_FILTER_SERIAL) {
        uint8_t *vis = calloc(n ? n : 1, 1), *qp = calloc(n ? n : 1, 1);
        orc_mark(&g, t, 0, n, tau_r, vis, qp, NULL);
        for (uint64_t i = 0; i < n; ++i) {
            const int cand = vis[i] && (qp[i] || t->leaf[i]);
            if (cand && !ancestor_disqualifies(t, (uint32_t)i, qp)) selected[ns++] = (uint32_t)i;
        }
        free(vis);
        free(qp);
        *passes = mode == ORC_FILTER_ORACLE ? 1 : 2;
        *barriers = mode == ORC_FILTER_ORACLE ? 0 : 2;
        *n_selected = ns;
        return ORC_OK;
    }
    /* serial: child adjacency as scene.cpp:74-82 (ascending child index per parent) */
    uint32_t *coff = calloc(n + 1, sizeof(uint32_t));
    for (uint64_t i = 0; i < n; ++i)
        if (t->parent[i] != ORC_ROOT_PARENT) ++coff[t->parent[i] + 1];
    for (uint64_t i = 1; i <= n; ++i) coff[i] += coff[i - 1];
    uint32_t *cidx = malloc((coff[n] ? coff[n] : 1) * sizeof(uint32_t));
    uint32_t *cur = malloc((n ? n : 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < n; ++i) cur[i] = coff[i];
    for (uint64_t i = 0; i < n; ++i)
        if (t->parent[i] != ORC_ROOT_PARENT) cidx[cur[t->parent[i]]++] = (uint32_t)i;
    uint32_t *active = malloc((n ? n : 1) * sizeof(uint32_t));
    uint32_t *next = malloc((n ? n : 1) * sizeof(uint32_t));
    uint64_t na = 0;
    const uint32_t l0_end = t->n_levels ? level_end(t, 0) : 0;
    for (uint32_t i = 0; i < l0_end; ++i) active[na++] = i;
    int p = 0, b = 0;
    orc_mark_out o;
    for (uint32_t level = 0; level < t->n_levels && na > 0; ++level) {
        ++p;
        ++b;
        uint64_t nn = 0;
        for (uint64_t i = 0; i < na; ++i) {
            const uint32_t idx = active[i];
            mark_node(&g, t, idx, tau_r, &o);
            if (!o.vis) continue;
            if (o.qpass || t->leaf[idx]) {
                selected[ns++] = idx;
            } else {
                for (uint32_t c = coff[idx]; c < coff[idx + 1]; ++c) next[nn++] = cidx[c];
            }
        }
        uint32_t *tmp = active;
        active = next;
        next = tmp;
        na = nn;
    }
    free(coff);
    free(cidx);
    free(cur);
    free(active);
    free(next);
    *passes = p;
    *barriers = b;
    *n_selected = ns;
    return ORC_OK;
}

/* -------------------------------------------------------- preprocessing -- */
/* projection.cpp:60-91. 1 projected, 0 culled, -1 non-finite (ValidationError). */
int orc_project(const orc_geom *g, const orc_tree *t, uint32_t idx, orc_proj *p) {
    orc_mark_out m;
    mark_node(g, t, idx, INFINITY, &m);
    if (!m.vis || !m.z_ok) return 0;
    p->node = idx;
    const double inv_z = 1.0 / m.tz;
    p->mean2d_x = g->fx * (m.tx * inv_z) + g->cx;
    p->mean2d_y = g->fy * (m.ty * inv_z) + g->cy;
    p->cov_a = m.a;
    p->cov_b = m.b;
    p->cov_c = m.c;
    const double det = m.a * m.c - m.b * m.b;
    p->conic_a = m.c / det;
    p->conic_b = -m.b / det;
    p->conic_c = m.a / det;
    p->sigma_max = sqrt(m.lambda_max);
    p->sigma_min = sqrt(m.lambda_min);
    p->depth = m.tz;
    p->radius = m.radius;
    const double v[12] = {p->mean2d_x, p->mean2d_y, p->cov_a,     p->cov_b,
                          p->cov_c,    p->conic_a,  p->conic_b,   p->conic_c,
                          p->sigma_max, p->sigma_min, p->depth, p->radius};
    for (int i = 0; i < 12; ++i)
        if (!isfinite(v[i])) return -1;
    return 1;
}

/* rasterizer.cpp:36-46 */
double orc_effective_radius(double sigma_max, float opacity, int kind, double tau, int *err) {
    const double three_sigma = 3.0 * sigma_max;
    if (err) *err = 0;
    if (kind == ORC_SHRINK_THREE_SIGMA) return three_sigma;
    if (!(tau > 0.0 && tau < 1.0)) {
        if (err) *err = ORC_EVALIDATION;
        return 0.0;
    }
    const double a0 = (double)opacity;
    if (a0 <= tau) return 0.0;
    const double r = sigma_max * sqrt(2.0 * log(a0 / tau));
    return smin(r, three_sigma);
}

/* rasterizer.cpp:48-73. Returns the number of gaussians, or -ORC_EVALIDATION. */
int orc_prepare(const orc_tree *t, const orc_camera *cam, const uint32_t *selected, uint64_t n_sel,
                int kind, double tau, orc_blendlist *out) {
    orc_geom g;
    orc_camera_geom(cam, &g);
    uint64_t k = 0;
    for (uint64_t s = 0; s < n_sel; ++s) {
        const uint32_t idx = selected[s];
        orc_proj p;
        const int rc = orc_project(&g, t, idx, &p);
        if (rc < 0) return -ORC_EVALIDATION;
        if (rc == 0) continue;
        int err = 0;
        const double r = orc_effective_radius(p.sigma_max, t->opacity[idx], kind, tau, &err);
        if (err) return -ORC_EVALIDATION;
        out->mean_x[k] = p.mean2d_x;
        out->mean_y[k] = p.mean2d_y;
        out->conic_a[k] = p.conic_a;
        out->conic_b[k] = p.conic_b;
        out->conic_c[k] = p.conic_c;
        out->opacity[k] = (double)t->opacity[idx];
        out->col_r[k] = (double)t->color_r[idx];
        out->col_g[k] = (double)t->color_g[idx];
        out->col_b[k] = (double)t->color_b[idx];
        out->radius[k] = r;
        out->depth[k] = (float)p.depth;
        out->node[k] = idx;
        ++k;
    }
    out->n = k;
    return (int)k;
}

/* ---------------------------------------------------------------- binning -- */
typedef struct {
    int tx0, tx1, ty0, ty1;
} rect_t;

/* rasterizer.cpp:78-91 */
static int tile_rect(double mx, double my, double r, int tiles_x, int tiles_y, rect_t *o) {
    if (!(r > 0.0)) return 0;
    int tx0 = (int)floor((mx - r) / ORC_TILE);
    int tx1 = (int)floor((mx + r) / ORC_TILE);
    int ty0 = (int)floor((my - r) / ORC_TILE);
    int ty1 = (int)floor((my + r) / ORC_TILE);
    o->tx0 = tx0 < 0 ? 0 : tx0;
    o->ty0 = ty0 < 0 ? 0 : ty0;
    o->tx1 = tx1 > tiles_x - 1 ? tiles_x - 1 : tx1;
    o->ty1 = ty1 > tiles_y - 1 ? tiles_y - 1 : ty1;
    return 1;
}

uint64_t orc_bin_count(const orc_blendlist *l, int width, int height) {
    const int tiles_x = (width + ORC_TILE - 1) / ORC_TILE, tiles_y = (height + ORC_TILE - 1) / ORC_TILE;
    uint64_t n = 0;
    for (uint64_t i = 0; i < l->n; ++i) {
        rect_t r;
        if (!tile_rect(l->mean_x[i], l->mean_y[i], l->radius[i], tiles_x, tiles_y, &r)) continue;
        if (r.tx1 < r.tx0 || r.ty1 < r.ty0) continue;
        n += (uint64_t)(r.tx1 - r.tx0 + 1) * (uint64_t)(r.ty1 - r.ty0 + 1);
    }
    return n;
}

/* rasterizer.cpp:75-98: row-major tiles per gaussian, gaussians in list order. */
uint64_t orc_bin_to_tiles(const orc_blendlist *l, int width, int height, orc_pair *out) {
    const int tiles_x = (width + ORC_TILE - 1) / ORC_TILE, tiles_y = (height + ORC_TILE - 1) / ORC_TILE;
    uint64_t k = 0;
    for (uint64_t i = 0; i < l->n; ++i) {
        rect_t r;
        if (!tile_rect(l->mean_x[i], l->mean_y[i], l->radius[i], tiles_x, tiles_y, &r)) continue;
        for (int ty = r.ty0; ty <= r.ty1; ++ty)
            for (int tx = r.tx0; tx <= r.tx1; ++tx) {
                out[k].tile = (uint32_t)ty * (uint32_t)tiles_x + (uint32_t)tx;
                out[k].depth = l->depth[i];
                out[k].gaussian = (uint32_t)i;
                ++k;
            }
    }
    return k;
}

/* ------------------------------------------------------------------ sort -- */
/* rasterizer.cpp:100-135: LSD radix over the packed (tile<<32 | depth bits)
 * key, one byte per pass, skipping passes whose digit is uniform. */
void orc_sort_pairs(orc_pair *pairs, uint64_t n) {
    if (n < 2) return;
    uint64_t *keys = malloc(n * 8), *keys_tmp = malloc(n * 8);
    uint32_t *order = malloc(n * 4), *order_tmp = malloc(n * 4);
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t bits;
        memcpy(&bits, &pairs[i].depth, 4);
        keys[i] = ((uint64_t)pairs[i].tile << 32) | bits;
        order[i] = (uint32_t)i;
    }
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = pass * 8;
        uint64_t count[256] = {0};
        for (uint64_t i = 0; i < n; ++i) ++count[(keys[i] >> shift) & 0xff];
        if (count[(keys[0] >> shift) & 0xff] == n) continue;
        uint64_t sum = 0;
        for (int b = 0; b < 256; ++b) {
            const uint64_t c = count[b];
            count[b] = sum;
            sum += c;
        }
        for (uint64_t i = 0; i < n; ++i) {
            const uint64_t dst = count[(keys[i] >> shift) & 0xff]++;
            keys_tmp[dst] = keys[i];
            order_tmp[dst] = order[i];
        }
        uint64_t *tk = keys;
        keys = keys_tmp;
        keys_tmp = tk;
        uint32_t *to = order;
        order = order_tmp;
        order_tmp = to;
    }
    orc_pair *sorted = malloc(n * sizeof(orc_pair));
    for (uint64_t i = 0; i < n; ++i) sorted[i] = pairs[order[i]];
    memcpy(pairs, sorted, n * sizeof(orc_pair));
    free(sorted);
    free(keys);
    free(keys_tmp);
    free(order);
    free(order_tmp);
}

/* ----------------------------------------------------------------- blend -- */
/* fastexp.hpp:18-50 */
static const double kExpPoly[13] = {1.0,
                                    1.0,
                                    1.0 / 2,
                                    1.0 / 6,
                                    1.0 / 24,
                                    1.0 / 120,
                                    1.0 / 720,
                                    1.0 / 5040,
                                    1.0 / 40320,
                                    1.0 / 362880,
                                    1.0 / 3628800,
                                    1.0 / 39916800,
                                    1.0 / 479001600};

double orc_exp_mx(double x) {
    x = smax(x, -30.0);
    const double t = x * 1.44269504088896338700e+00;
    const double u = t + 6755399441055744.0;
    const double fn = u - 6755399441055744.0;
    const double r1 = x - fn * 6.93147180369123816490e-01;
    const double r = r1 - fn * 1.90821492927058770002e-10;
    double p = kExpPoly[12];
    for (int k = 11; k >= 0; --k) p = p * r + kExpPoly[k];
    const int64_t n = (int64_t)fn;
    const uint64_t bits = (uint64_t)(n + 1023) << 52;
    double scale;
    memcpy(&scale, &bits, 8);
    return p * scale;
}

#define K_ALPHA_CAP 0.99          /* kernels.hpp:20 */
#define K_MIN_ALPHA (1.0 / 255.0) /* kernels.hpp:21 */
#define K_TERM_T 1e-4             /* kernels.hpp:22 */

/* blend_scalar.cpp:13-55, including the 4-lane kpc partials. */
void orc_blend_tile(const orc_blendlist *g, const orc_pair *pairs, uint64_t n_pairs, int x0,
                    int y0, int w, int h, int img_w, float *image, double *kpc_out) {
    double *acc = kpc_out ? calloc(n_pairs * 4 + 1, sizeof(double)) : NULL;
    for (int y = y0; y < y0 + h; ++y) {
        const double py = (double)y + 0.5;
        for (int x = x0; x < x0 + w; ++x) {
            const double px = (double)x + 0.5;
            const int lane = (x - x0) & 3;
            double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0;
            for (uint64_t j = 0; j < n_pairs; ++j) {
                const uint32_t k = pairs[j].gaussian;
                const double dx = px - g->mean_x[k];
                const double dy = py - g->mean_y[k];
                const double t1 = (g->conic_a[k] * dx) * dx;
                const double t2 = (g->conic_c[k] * dy) * dy;
                const double t3 = (g->conic_b[k] * dx) * dy;
                const double power = -0.5 * (t1 + t2) - t3;
                const double alpha = smin(g->opacity[k] * orc_exp_mx(power), K_ALPHA_CAP);
                if (alpha < K_MIN_ALPHA) continue;
                const double wgt = alpha * T;
                cr += g->col_r[k] * wgt;
                cg += g->col_g[k] * wgt;
                cb += g->col_b[k] * wgt;
                if (acc) acc[j * 4 + lane] += wgt;
                T *= 1.0 - alpha;
                if (T < K_TERM_T) break;
            }
            float *o = image + ((size_t)y * img_w + x) * 3;
            o[0] = (float)cr;
            o[1] = (float)cg;
            o[2] = (float)cb;
        }
    }
    if (acc) {
        for (uint64_t j = 0; j < n_pairs; ++j)
            kpc_out[j] = (acc[j * 4 + 0] + acc[j * 4 + 1]) + (acc[j * 4 + 2] + acc[j * 4 + 3]);
        free(acc);
    }
}

/* rasterizer.cpp:137-165 */
int orc_alpha_blend(const orc_pair *sorted, uint64_t n, const orc_blendlist *l, int width,
                    int height, float *image, double *kpc_out) {
    const int tiles_x = (width + ORC_TILE - 1) / ORC_TILE, tiles_y = (height + ORC_TILE - 1) / ORC_TILE;
    const uint64_t n_tile = (uint64_t)tiles_x * tiles_y;
    memset(image, 0, (size_t)width * height * 3 * sizeof(float));
    uint64_t *off = calloc(n_tile + 1, sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) ++off[sorted[i].tile + 1];
    for (uint64_t t = 0; t < n_tile; ++t) off[t + 1] += off[t];
    if (kpc_out)
        for (uint64_t i = 0; i < n; ++i) kpc_out[i] = 0.0;
    for (uint64_t t = 0; t < n_tile; ++t) {
        const uint64_t b = off[t], e = off[t + 1];
        if (b == e) continue;
        const int tx = (int)t % tiles_x, ty = (int)t / tiles_x;
        const int x0 = tx * ORC_TILE, y0 = ty * ORC_TILE;
        const int w = ORC_TILE < width - x0 ? ORC_TILE : width - x0;
        const int h = ORC_TILE < height - y0 ? ORC_TILE : height - y0;
        orc_blend_tile(l, sorted + b, e - b, x0, y0, w, h, width, image,
                       kpc_out ? kpc_out + b : NULL);
    }
    free(off);
    return ORC_OK;
}

/* ---------------------------------------------------------------- render -- */
struct orc_render_out {
    orc_stats st;
    float *image;
    uint32_t *selected;
    orc_pair *pairs;
    double *kpc;
    orc_blendlist list;
    void *list_mem;
};

static void blendlist_alloc(orc_blendlist *l, uint64_t cap, void **mem) {
    if (cap == 0) cap = 1;
    char *m = malloc(cap * (10 * 8 + 4 + 4));
    *mem = m;
    double **f[10] = {&l->mean_x, &l->mean_y, &l->conic_a, &l->conic_b, &l->conic_c,
                      &l->opacity, &l->col_r, &l->col_g, &l->col_b, &l->radius};
    for (int i = 0; i < 10; ++i) *f[i] = (double *)(m + (size_t)i * cap * 8);
    l->depth = (float *)(m + 10 * cap * 8);
    l->node = (uint32_t *)(m + 10 * cap * 8 + cap * 4);
    l->n = 0;
}

/* rasterizer.cpp:167-213 (validation of the tree itself is the caller's job). */
orc_render_out *orc_render(const orc_tree *t, const orc_camera *cam, double tau_r, int kind,
                           double tau, int collect_kpc, int *err) {
    *err = 0;
    if (kind != ORC_SHRINK_THREE_SIGMA && !(tau > 0.0 && tau < 1.0)) {
        *err = ORC_EVALIDATION;
        return NULL;
    }
    orc_render_out *r = calloc(1, sizeof *r);
    r->selected = malloc((t->n ? t->n : 1) * 4);
    uint64_t ns = 0;
    int rc = orc_filter(t, cam, tau_r, ORC_FILTER_PARALLEL, r->selected, &ns, &r->st.passes,
                        &r->st.barriers);
    if (rc) {
        *err = rc;
        orc_render_free(r);
        return NULL;
    }
    r->st.n_selected = ns;
    blendlist_alloc(&r->list, ns, &r->list_mem);
    const int ng = orc_prepare(t, cam, r->selected, ns, kind, tau, &r->list);
    if (ng < 0) {
        *err = -ng;
        orc_render_free(r);
        return NULL;
    }
    r->st.n_gaussians = (uint64_t)ng;
    const uint64_t np = orc_bin_count(&r->list, cam->width, cam->height);
    r->pairs = malloc((np ? np : 1) * sizeof(orc_pair));
    orc_bin_to_tiles(&r->list, cam->width, cam->height, r->pairs);
    r->st.n_pairs = np;
    orc_sort_pairs(r->pairs, np);
    r->image = malloc((size_t)cam->width * cam->height * 3 * sizeof(float));
    if (collect_kpc) r->kpc = malloc((np ? np : 1) * sizeof(double));
    orc_alpha_blend(r->pairs, np, &r->list, cam->width, cam->height, r->image, r->kpc);
    return r;
}

void orc_render_stats(const orc_render_out *r, orc_stats *st) { *st = r->st; }
const float *orc_render_image(const orc_render_out *r) { return r->image; }
const orc_pair *orc_render_pairs(const orc_render_out *r) { return r->pairs; }
const double *orc_render_kpc(const orc_render_out *r) { return r->kpc; }
const uint32_t *orc_render_selected(const orc_render_out *r) { return r->selected; }
void orc_render_gaussians(const orc_render_out *r, orc_blendlist *out) { *out = r->list; }
void orc_render_free(orc_render_out *r) {
    if (!r) return;
    free(r->image);
    free(r->selected);
    free(r->pairs);
    free(r->kpc);
    free(r->list_mem);
    free(r);
}

/* --------------------------------------------------------------- metrics -- */
/* metrics.cpp:18-42 */
double orc_view_gtc(const orc_pair *sorted, const double *kpc, uint64_t n) {
    if (n == 0) return NAN;
    double sum_tiles = 0.0;
    uint64_t n_tiles = 0, i = 0;
    while (i < n) {
        const uint32_t tile = sorted[i].tile;
        double sum = 0.0;
        uint32_t c = 0;
        for (; i < n && sorted[i].tile == tile; ++i) {
            sum += kpc[i];
            ++c;
        }
        sum_tiles += sum / (double)c;
        ++n_tiles;
    }
    return sum_tiles / (double)n_tiles;
}

/* metrics.cpp:121-132 */
double orc_psnr(const float *a, const float *b, uint64_t n) {
    double se = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double d = (double)a[i] - (double)b[i];
        se += d * d;
    }
    const double mse = se / (double)n;
    if (mse == 0.0) return INFINITY;
    return 10.0 * log10(1.0 / mse);
}

/* metrics.cpp:44-57 */
void orc_redundancy_histogram(const double *kpc, uint64_t n, uint64_t bins[5]) {
    static const double edges[4] = {0.01, 0.05, 0.2, 1.0};
    for (int i = 0; i < 5; ++i) bins[i] = 0;
    for (uint64_t i = 0; i < n; ++i) {
        int b = 4;
        for (int e = 0; e < 4; ++e)
            if (kpc[i] < edges[e]) {
                b = e;
                break;
            }
        ++bins[b];
    }
}
