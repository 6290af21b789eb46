/* lodgs_oracle.h -- TEST INFRASTRUCTURE ONLY: the CPU checker, never the product.
 *
 * Plain-C restatement of the reference per-frame render path
 * (/root/reference/proj, the `lodgs` C++20 library).  Each function cites the
 * reference file:line it restates.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load oracle/_build/liboracle.so.
 *
 * Parity pinning: tests/test_oracle_cpu.py checks every function here against
 * the reference library compiled in place (oracle/_ref, see oracle/Makefile) and
 * against the reference's own known-answer tests restated in tests/golden/.
 *
 * Floating point: compiled with -ffp-contract=off (as the reference,
 * proj/CMakeLists.txt:13), same association as mark_core.hpp:24-116.
 */
#ifndef LODGS_ORACLE_H
#define LODGS_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_ROOT_PARENT 0xFFFFFFFFu /* core.hpp:15 kRootParent */
#define ORC_TILE 16                  /* tiles.hpp:8-9 */

/* scene.hpp:76-82 Camera (same memory layout as lodgs_camera in include/lodgs_gpu.h) */
typedef struct {
    uint32_t width, height;
    double fx, fy, cx, cy;
    double rotation[9];    /* world->camera, row-major */
    double translation[3];
    double znear, zfar;
} orc_camera;

/* projection.hpp:23-32 CameraGeom (44 doubles) */
typedef struct {
    double rot[9];
    double trans[3];
    double fx, fy, cx, cy;
    double width, height;
    double znear, zfar;
    double planes[6][4];
} orc_geom;

/* scene.hpp:29-74 LoDTree as raw SoA views */
typedef struct {
    uint64_t n;
    const float *mean_x, *mean_y, *mean_z;
    const float *scale_x, *scale_y, *scale_z;
    const float *quat_w, *quat_x, *quat_y, *quat_z;
    const float *opacity;
    const float *color_r, *color_g, *color_b;
    const uint32_t *parent;
    const uint8_t *leaf;
    const uint32_t *level_offsets;
    uint32_t n_levels;
} orc_tree;

/* tiles.hpp:23-28 TilePair */
typedef struct {
    uint32_t tile;
    float depth;
    uint32_t gaussian;
} orc_pair;

/* rasterizer.hpp:36-51 BlendList, caller-owned arrays of capacity >= n */
typedef struct {
    uint64_t n;
    double *mean_x, *mean_y, *conic_a, *conic_b, *conic_c, *opacity, *col_r, *col_g, *col_b,
        *radius;
    float *depth;
    uint32_t *node;
} orc_blendlist;

typedef struct {
    double tx, ty, tz, a, b, c, lambda_max, lambda_min, radius;
    int vis, z_ok, qpass;
} orc_mark_out;

typedef struct {
    double mean2d_x, mean2d_y, cov_a, cov_b, cov_c, conic_a, conic_b, conic_c, sigma_max,
        sigma_min, depth, radius;
    uint32_t node;
} orc_proj;

enum { ORC_SHRINK_THREE_SIGMA = 0, ORC_SHRINK_FIXED = 1, ORC_SHRINK_ADAPTIVE = 2 };
enum { ORC_FILTER_ORACLE = 0, ORC_FILTER_SERIAL = 1, ORC_FILTER_PARALLEL = 2 };
enum { ORC_OK = 0, ORC_EVALIDATION = 2 };

typedef struct {
    uint64_t n_selected, n_pairs, n_gaussians;
    int32_t passes, barriers;
} orc_stats;

/* ---- rng.hpp:11-33 (mt19937_64 + splitmix finaliser) ---- */
typedef struct {
    uint64_t mt[312];
    int idx;
} orc_rng;
void orc_rng_seed(orc_rng *r, uint64_t seed);
uint64_t orc_rng_next_u64(orc_rng *r);
double orc_rng_next_double(orc_rng *r);
double orc_rng_uniform(orc_rng *r, double lo, double hi);
uint64_t orc_rng_next_below(orc_rng *r, uint64_t n);
uint64_t orc_mix_seed(uint64_t seed, uint64_t item);
size_t orc_rng_sizeof(void);

/* ---- tests/unit/test_util.hpp:19-60 camera fixtures ---- */
void orc_front_camera(uint32_t w, uint32_t h, double focal, orc_camera *out);
void orc_orbit_camera(orc_rng *r, uint32_t w, uint32_t h, double dist, orc_camera *out);

/* ---- projection.cpp:11-38, mark_core.hpp:24-116 ---- */
void orc_camera_geom(const orc_camera *cam, orc_geom *g);
void orc_mark_core(const orc_geom *g, float mx, float my, float mz, float sx, float sy, float sz,
                   float qw, float qx, float qy, float qz, double tau_r, orc_mark_out *o);
/* mark_scalar.cpp:7-19 */
void orc_mark(const orc_geom *g, const orc_tree *t, uint64_t begin, uint64_t end, double tau_r,
              uint8_t *vis, uint8_t *qpass, double *radius_out);

/* ---- filter.cpp:29-150 ---- */
int orc_filter(const orc_tree *t, const orc_camera *cam, double tau_r, int mode,
               uint32_t *selected /* cap t->n */, uint64_t *n_selected, int32_t *passes,
               int32_t *barriers);

/* ---- projection.cpp:60-91, rasterizer.cpp:36-73 ---- */
int orc_project(const orc_geom *g, const orc_tree *t, uint32_t idx, orc_proj *p); /* 1 ok, 0 culled, -1 non-finite */
double orc_effective_radius(double sigma_max, float opacity, int kind, double tau, int *err);
int orc_prepare(const orc_tree *t, const orc_camera *cam, const uint32_t *selected, uint64_t n_sel,
                int kind, double tau, orc_blendlist *out);

/* ---- rasterizer.cpp:75-165 ---- */
uint64_t orc_bin_count(const orc_blendlist *l, int width, int height);
uint64_t orc_bin_to_tiles(const orc_blendlist *l, int width, int height, orc_pair *out);
void orc_sort_pairs(orc_pair *pairs, uint64_t n);
double orc_exp_mx(double x); /* fastexp.hpp:38-50 */
void orc_blend_tile(const orc_blendlist *g, const orc_pair *pairs, uint64_t n_pairs, int x0,
                    int y0, int w, int h, int img_w, float *image, double *kpc_out);
int orc_alpha_blend(const orc_pair *sorted, uint64_t n, const orc_blendlist *l, int width,
                    int height, float *image /* w*h*3 */, double *kpc_out /* n or NULL */);

/* ---- rasterizer.cpp:167-213: whole frame. Result owned by the handle. ---- */
typedef struct orc_render_out orc_render_out;
orc_render_out *orc_render(const orc_tree *t, const orc_camera *cam, double tau_r, int kind,
                           double tau, int collect_kpc, int *err);
void orc_render_stats(const orc_render_out *r, orc_stats *st);
const float *orc_render_image(const orc_render_out *r);
const orc_pair *orc_render_pairs(const orc_render_out *r);
const double *orc_render_kpc(const orc_render_out *r);
const uint32_t *orc_render_selected(const orc_render_out *r);
void orc_render_gaussians(const orc_render_out *r, orc_blendlist *out);
void orc_render_free(orc_render_out *r);

/* ---- metrics.cpp:18-132 ---- */
double orc_view_gtc(const orc_pair *sorted, const double *kpc, uint64_t n);
double orc_psnr(const float *a, const float *b, uint64_t n_floats);
void orc_redundancy_histogram(const double *kpc, uint64_t n, uint64_t bins5[5]);

#ifdef __cplusplus
}
#endif
#endif
