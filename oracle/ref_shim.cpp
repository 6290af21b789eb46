// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A flat extern "C" surface over the *unmodified* reference library
// (/root/reference/proj, compiled in place by oracle/Makefile into
// oracle/_ref/libref_lodgs.so).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load it.  Nothing in the
// product (paper_2603_23891_b200/) links or calls this.
//
// Every entry point forwards to the reference symbol named in its comment;
// no algorithmic code lives here.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "lodgs/camera_path.hpp"
#include "lodgs/filter.hpp"
#include "lodgs/kernels.hpp"
#include "lodgs/metrics.hpp"
#include "lodgs/projection.hpp"
#include "lodgs/rasterizer.hpp"
#include "lodgs/rng.hpp"
#include "lodgs/scene.hpp"
#include "lodgs/tree_builder.hpp"
#include "kernels/fastexp.hpp"
#include "../tests/unit/test_util.hpp"

using namespace lodgs;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ValidationError*>(&e)) return 2;
    return 1;
}
}  // namespace

extern "C" {

// Camera POD shared with the Python side (same layout as lodgs_camera in
// include/lodgs_gpu.h).
struct ref_camera {
    uint32_t width, height;
    double fx, fy, cx, cy;
    double rotation[9];
    double translation[3];
    double znear, zfar;
};

static Camera to_cam(const ref_camera* c) {
    Camera k;
    k.width = c->width;
    k.height = c->height;
    k.fx = c->fx;
    k.fy = c->fy;
    k.cx = c->cx;
    k.cy = c->cy;
    for (int i = 0; i < 9; ++i) k.world_to_cam_rotation[i] = c->rotation[i];
    for (int i = 0; i < 3; ++i) k.world_to_cam_translation[i] = c->translation[i];
    k.near = c->znear;
    k.far = c->zfar;
    return k;
}

static void from_cam(const Camera& k, ref_camera* c) {
    c->width = k.width;
    c->height = k.height;
    c->fx = k.fx;
    c->fy = k.fy;
    c->cx = k.cx;
    c->cy = k.cy;
    for (int i = 0; i < 9; ++i) c->rotation[i] = k.world_to_cam_rotation[i];
    for (int i = 0; i < 3; ++i) c->translation[i] = k.world_to_cam_translation[i];
    c->znear = k.near;
    c->zfar = k.far;
}

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- trees --
// tests/unit/test_util.hpp:62-77 (test::make_tree)
void* ref_make_tree(uint64_t seed, uint32_t depth, uint32_t children, float gamma,
                    uint32_t nx, uint32_t ny, uint32_t congestion) {
    try {
        return new LoDTree(test::make_tree(seed, depth, children, gamma, nx, ny,
                                           congestion));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// tree_builder.cpp:126-174 + :75-124 with every spec field exposed.
void* ref_build_synthetic(uint32_t nx, uint32_t ny, float spacing, float scale_min,
                          float scale_max, float opacity_min, float opacity_max,
                          uint64_t scene_seed, uint32_t congestion, uint32_t depth,
                          float shrink, uint32_t children, uint64_t build_seed) {
    try {
        SyntheticSceneSpec s;
        s.nx = nx;
        s.ny = ny;
        s.spacing = spacing;
        s.scale_min = scale_min;
        s.scale_max = scale_max;
        s.opacity_min = opacity_min;
        s.opacity_max = opacity_max;
        s.seed = scene_seed;
        s.congestion = congestion;
        TreeBuildConfig c;
        c.depth = depth;
        c.shrink_factor = shrink;
        c.children_per_node = children;
        c.seed = build_seed;
        return new LoDTree(build_tree(generate_synthetic_scene(s), c));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// Builds a LoDTree from raw SoA arrays (hand KAT fixtures); scene.cpp:64-82.
void* ref_tree_from_arrays(uint64_t n, const float* const* fields14,
                           const uint32_t* parent, const uint8_t* leaf,
                           const uint32_t* level_offsets, uint32_t n_levels,
                           float shrink) {
    auto* t = new LoDTree();
    std::vector<float>* f[14] = {&t->mean_x,  &t->mean_y,  &t->mean_z,  &t->scale_x,
                                 &t->scale_y, &t->scale_z, &t->quat_w,  &t->quat_x,
                                 &t->quat_y,  &t->quat_z,  &t->opacity, &t->color_r,
                                 &t->color_g, &t->color_b};
    for (int k = 0; k < 14; ++k) f[k]->assign(fields14[k], fields14[k] + n);
    t->parent.assign(parent, parent + n);
    t->leaf.assign(leaf, leaf + n);
    t->level_offsets.assign(level_offsets, level_offsets + n_levels);
    t->shrink_factor = shrink;
    t->rebuild_derived();
    return t;
}

uint64_t ref_tree_size(void* h) { return static_cast<LoDTree*>(h)->node_count(); }
uint32_t ref_tree_levels(void* h) {
    return uint32_t(static_cast<LoDTree*>(h)->level_count());
}

void ref_tree_export(void* h, float* const* fields14, uint32_t* parent, uint8_t* leaf,
                     uint32_t* level_offsets) {
    const LoDTree& t = *static_cast<LoDTree*>(h);
    const std::vector<float>* f[14] = {&t.mean_x,  &t.mean_y,  &t.mean_z,  &t.scale_x,
                                       &t.scale_y, &t.scale_z, &t.quat_w,  &t.quat_x,
                                       &t.quat_y,  &t.quat_z,  &t.opacity, &t.color_r,
                                       &t.color_g, &t.color_b};
    for (int k = 0; k < 14; ++k)
        std::memcpy(fields14[k], f[k]->data(), f[k]->size() * sizeof(float));
    std::memcpy(parent, t.parent.data(), t.parent.size() * 4);
    std::memcpy(leaf, t.leaf.data(), t.leaf.size());
    std::memcpy(level_offsets, t.level_offsets.data(), t.level_offsets.size() * 4);
}

void ref_tree_free(void* h) { delete static_cast<LoDTree*>(h); }

// scene.cpp:89-165
uint64_t ref_validate_tree(void* h) {
    return validate_tree(*static_cast<LoDTree*>(h)).size();
}

// --------------------------------------------------------------- rng --
// rng.hpp:11-33
void* ref_rng_new(uint64_t seed) { return new Rng(seed); }
void ref_rng_free(void* r) { delete static_cast<Rng*>(r); }
uint64_t ref_rng_next_u64(void* r) { return static_cast<Rng*>(r)->next_u64(); }
double ref_rng_uniform(void* r, double lo, double hi) {
    return static_cast<Rng*>(r)->uniform(lo, hi);
}
uint64_t ref_rng_next_below(void* r, uint64_t n) {
    return static_cast<Rng*>(r)->next_below(n);
}
uint64_t ref_mix_seed(uint64_t s, uint64_t i) { return mix_seed(s, i); }

// test_util.hpp:19-60
void ref_orbit_camera(void* r, uint32_t w, uint32_t h, double dist, ref_camera* out) {
    from_cam(test::orbit_camera(*static_cast<Rng*>(r), w, h, dist), out);
}
void ref_front_camera(uint32_t w, uint32_t h, double focal, ref_camera* out) {
    from_cam(test::front_camera(w, h, focal), out);
}

// camera_path.cpp:126-193
int ref_camera_path_sample(const ref_camera* keys, uint32_t n_keys,
                           const uint32_t* samples, ref_camera* out) {
    try {
        CameraPath p;
        for (uint32_t i = 0; i < n_keys; ++i) p.keyframes.push_back(to_cam(&keys[i]));
        for (uint32_t i = 0; i + 1 < n_keys; ++i) p.samples.push_back(samples[i]);
        const auto frames = p.sample();
        for (std::size_t i = 0; i < frames.size(); ++i) from_cam(frames[i], &out[i]);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// projection.cpp:11-38
void ref_camera_geom(const ref_camera* c, double* out44) {
    const CameraGeom g = CameraGeom::make(to_cam(c));
    std::memcpy(out44, &g, sizeof(CameraGeom));
}

// ------------------------------------------------------------- kernels --
// kernels.hpp:47-52 via the active KernelTable (scalar or avx2).
int ref_mark(void* h, const ref_camera* c, uint64_t begin, uint64_t end, double tau_r,
             uint8_t* vis, uint8_t* qpass, double* radius, int backend) {
    try {
        if (backend == 0) force_kernel_backend(Backend::scalar);
        else if (backend == 1) force_kernel_backend(Backend::avx2);
        const LoDTree& t = *static_cast<LoDTree*>(h);
        kernels().mark(CameraGeom::make(to_cam(c)), NodeArrays::from(t), begin, end,
                       tau_r, vis, qpass, radius);
        reset_kernel_backend();
        return 0;
    } catch (const std::exception& e) {
        reset_kernel_backend();
        return fail(e);
    }
}

// fastexp.hpp:38-50
double ref_exp_mx(double x) { return detail::exp_mx(x); }

// rasterizer.cpp:36-46
double ref_effective_radius(double sigma_max, float opacity, int kind, double tau) {
    Projected2D p;
    p.sigma_max = sigma_max;
    p.radius = 3.0 * sigma_max;
    ShrinkMode m{ShrinkMode::Kind(kind), tau};
    try {
        return effective_radius(p, opacity, m);
    } catch (const std::exception& e) {
        fail(e);
        return -1.0;
    }
}

// filter.cpp:29-150; mode 0 oracle, 1 serial, 2 parallel.
int ref_filter(void* h, const ref_camera* c, double tau_r, uint32_t workers, int mode,
               uint32_t* selected, uint64_t cap, uint64_t* n_out, int32_t* passes,
               int32_t* barriers, double* calc_ms, double* sync_ms) {
    try {
        const LoDTree& t = *static_cast<LoDTree*>(h);
        FilterConfig fc{tau_r, workers};
        FilterResult r = mode == 0   ? filter_oracle(t, to_cam(c), fc)
                         : mode == 1 ? filter_serial(t, to_cam(c), fc)
                                     : filter_parallel(t, to_cam(c), fc);
        *n_out = r.selected.size();
        if (r.selected.size() > cap) {
            g_err = "selected capacity";
            return 1;
        }
        std::memcpy(selected, r.selected.data(), r.selected.size() * 4);
        *passes = r.passes;
        *barriers = r.barriers;
        if (calc_ms) *calc_ms = r.calc_ms;
        if (sync_ms) *sync_ms = r.sync_ms;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ------------------------------------------------------ stage functions --
struct ref_blendlist_view {
    uint64_t n;
    double *mean_x, *mean_y, *conic_a, *conic_b, *conic_c, *opacity, *col_r, *col_g,
        *col_b, *radius;
    float* depth;
    uint32_t* node;
};

static BlendList to_list(const ref_blendlist_view* v) {
    BlendList l;
    const uint64_t n = v->n;
    l.mean_x.assign(v->mean_x, v->mean_x + n);
    l.mean_y.assign(v->mean_y, v->mean_y + n);
    l.conic_a.assign(v->conic_a, v->conic_a + n);
    l.conic_b.assign(v->conic_b, v->conic_b + n);
    l.conic_c.assign(v->conic_c, v->conic_c + n);
    l.opacity.assign(v->opacity, v->opacity + n);
    l.col_r.assign(v->col_r, v->col_r + n);
    l.col_g.assign(v->col_g, v->col_g + n);
    l.col_b.assign(v->col_b, v->col_b + n);
    l.radius.assign(v->radius, v->radius + n);
    l.depth.assign(v->depth, v->depth + n);
    l.node.assign(v->node, v->node + n);
    return l;
}

static void from_list(const BlendList& l, ref_blendlist_view* v) {
    const uint64_t n = l.size();
    v->n = n;
    std::memcpy(v->mean_x, l.mean_x.data(), n * 8);
    std::memcpy(v->mean_y, l.mean_y.data(), n * 8);
    std::memcpy(v->conic_a, l.conic_a.data(), n * 8);
    std::memcpy(v->conic_b, l.conic_b.data(), n * 8);
    std::memcpy(v->conic_c, l.conic_c.data(), n * 8);
    std::memcpy(v->opacity, l.opacity.data(), n * 8);
    std::memcpy(v->col_r, l.col_r.data(), n * 8);
    std::memcpy(v->col_g, l.col_g.data(), n * 8);
    std::memcpy(v->col_b, l.col_b.data(), n * 8);
    std::memcpy(v->radius, l.radius.data(), n * 8);
    std::memcpy(v->depth, l.depth.data(), n * 4);
    std::memcpy(v->node, l.node.data(), n * 4);
}

// rasterizer.cpp:48-73. Output arrays must hold n_sel entries.
int ref_prepare(void* h, const ref_camera* c, const uint32_t* selected, uint64_t n_sel,
                int kind, double tau, ref_blendlist_view* out) {
    try {
        std::vector<NodeIndex> sel(selected, selected + n_sel);
        const BlendList l = prepare_gaussians(*static_cast<LoDTree*>(h), to_cam(c), sel,
                                              ShrinkMode{ShrinkMode::Kind(kind), tau});
        from_list(l, out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// rasterizer.cpp:75-98. Pairs are returned through a handle (count unknown).
void* ref_bin_to_tiles(const ref_blendlist_view* v, int w, int h, uint64_t* n_pairs) {
    auto* p = new std::vector<TilePair>(
        bin_to_tiles(to_list(v), TileGrid::make(w, h), w, h));
    *n_pairs = p->size();
    return p;
}

void ref_pairs_copy(void* p, uint32_t* out_triples) {
    const auto& v = *static_cast<std::vector<TilePair>*>(p);
    std::memcpy(out_triples, v.data(), v.size() * sizeof(TilePair));
}
void ref_pairs_free(void* p) { delete static_cast<std::vector<TilePair>*>(p); }

// rasterizer.cpp:100-135, in place on packed {tile, depth, gaussian} triples.
void ref_sort_pairs(uint32_t* triples, uint64_t n) {
    std::vector<TilePair> v(n);
    std::memcpy(v.data(), triples, n * sizeof(TilePair));
    sort_pairs(v);
    std::memcpy(triples, v.data(), n * sizeof(TilePair));
}

// rasterizer.cpp:137-165
int ref_alpha_blend(const uint32_t* sorted_triples, uint64_t n, const ref_blendlist_view* v,
                    int w, int h, uint32_t workers, float* image, double* kpc) {
    try {
        std::vector<TilePair> s(n);
        std::memcpy(s.data(), sorted_triples, n * sizeof(TilePair));
        std::vector<double> k;
        const Image img = alpha_blend(s, to_list(v), TileGrid::make(w, h), w, h, workers,
                                      kpc ? &k : nullptr);
        std::memcpy(image, img.rgb.data(), img.rgb.size() * 4);
        if (kpc) std::memcpy(kpc, k.data(), k.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---------------------------------------------------------------- render --
struct ref_stats {
    uint64_t n_selected, n_pairs, n_gaussians;
    int32_t passes, barriers;
    double t_calc_ms, t_sync_ms, t_prepr_ms, t_sort_ms, t_alpha_ms;
};

// rasterizer.cpp:167-213. Returns a RenderOutput handle.
void* ref_render(void* h, const ref_camera* c, double tau_r, int kind, double tau,
                 uint32_t workers, int filter_mode, int collect_kpc, ref_stats* st) {
    try {
        RenderOptions o;
        o.worker_count = workers;
        o.collect_kpc = collect_kpc != 0;
        o.filter_mode = filter_mode == 1 ? FilterMode::serial : FilterMode::parallel;
        auto* out = new RenderOutput(render(*static_cast<LoDTree*>(h), to_cam(c),
                                            FilterConfig{tau_r, workers},
                                            ShrinkMode{ShrinkMode::Kind(kind), tau}, o));
        st->n_selected = out->stats.n_selected;
        st->n_pairs = out->stats.n_pairs;
        st->n_gaussians = out->gaussians.size();
        st->passes = out->stats.filter_passes;
        st->barriers = out->stats.filter_barriers;
        st->t_calc_ms = out->stats.t_calc_ms;
        st->t_sync_ms = out->stats.t_sync_ms;
        st->t_prepr_ms = out->stats.t_prepr_ms;
        st->t_sort_ms = out->stats.t_sort_ms;
        st->t_alpha_ms = out->stats.t_alpha_ms;
        return out;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_render_image(void* r, float* out) {
    const auto& o = *static_cast<RenderOutput*>(r);
    std::memcpy(out, o.image.rgb.data(), o.image.rgb.size() * 4);
}
void ref_render_pairs(void* r, uint32_t* triples, double* kpc) {
    const auto& o = *static_cast<RenderOutput*>(r);
    std::memcpy(triples, o.pairs.data(), o.pairs.size() * sizeof(TilePair));
    if (kpc) std::memcpy(kpc, o.kpc.data(), o.kpc.size() * 8);
}
void ref_render_gaussians(void* r, ref_blendlist_view* v) {
    from_list(static_cast<RenderOutput*>(r)->gaussians, v);
}
void ref_render_free(void* r) { delete static_cast<RenderOutput*>(r); }

// metrics.cpp:94-108
int ref_calibrate(void* h, const ref_camera* views, uint32_t n_views, double lambda_g,
                  double tau_r, uint32_t workers, double* tau_out, double* scene_gtc,
                  double* per_view, uint32_t* n_used, uint64_t* hist5) {
    try {
        std::vector<Camera> v;
        for (uint32_t i = 0; i < n_views; ++i) v.push_back(to_cam(&views[i]));
        const CalibrationReport r =
            calibrate(*static_cast<LoDTree*>(h), v, lambda_g, FilterConfig{tau_r, workers});
        *tau_out = r.tau;
        *scene_gtc = r.scene_mean;
        *n_used = r.n_views;
        for (std::size_t i = 0; i < r.per_view.size(); ++i) per_view[i] = r.per_view[i];
        for (int i = 0; i < 5; ++i) hist5[i] = r.histogram.bins[i];
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// metrics.cpp:18-42 on literal inputs.
double ref_view_gtc(const uint32_t* sorted_triples, const double* kpc, uint64_t n) {
    std::vector<TilePair> s(n);
    std::memcpy(s.data(), sorted_triples, n * sizeof(TilePair));
    return view_gtc(tile_stats_from(s, std::vector<double>(kpc, kpc + n)));
}

// metrics.cpp:121-132
double ref_psnr(const float* a, const float* b, int w, int h) {
    Image x{w, h, std::vector<float>(a, a + std::size_t(w) * h * 3)};
    Image y{w, h, std::vector<float>(b, b + std::size_t(w) * h * 3)};
    return psnr(x, y);
}

// metrics.cpp:136-192
double ref_ssim(const float* a, const float* b, int w, int h) {
    Image x{w, h, std::vector<float>(a, a + std::size_t(w) * h * 3)};
    Image y{w, h, std::vector<float>(b, b + std::size_t(w) * h * 3)};
    try {
        return ssim(x, y);
    } catch (const std::exception&) {
        return -1e300;
    }
}

}  // extern "C"
