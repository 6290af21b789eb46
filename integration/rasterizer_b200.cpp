// proj/src/rasterizer_b200.cpp  (maintainer-added; link -llodgs_b200)
#include <mutex>
#include "lodgs/rasterizer.hpp"
#include "lodgs_gpu.h"

namespace lodgs {
namespace {
[[noreturn]] void rethrow(int rc) {
    const std::string msg = lodgs_gpu_last_error();
    if (rc == LODGS_ERR_VALIDATION) throw ValidationError(msg);
    if (rc == LODGS_ERR_IO) throw IoError(msg);
    throw std::runtime_error(msg);
}
lodgs_tree_view view_of(const LoDTree& t) {
    return {t.node_count(), t.mean_x.data(), t.mean_y.data(), t.mean_z.data(),
            t.scale_x.data(), t.scale_y.data(), t.scale_z.data(), t.quat_w.data(),
            t.quat_x.data(), t.quat_y.data(), t.quat_z.data(), t.opacity.data(),
            t.color_r.data(), t.color_g.data(), t.color_b.data(), t.parent.data(),
            t.leaf.data(), t.level_offsets.data(), uint32_t(t.level_count()), t.shrink_factor};
}
lodgs_camera cam_of(const Camera& c) {
    lodgs_camera k{c.width, c.height, c.fx, c.fy, c.cx, c.cy, {}, {}, c.near, c.far};
    for (int i = 0; i < 9; ++i) k.rotation[i] = c.world_to_cam_rotation[i];
    for (int i = 0; i < 3; ++i) k.translation[i] = c.world_to_cam_translation[i];
    return k;
}
// The tree is immutable while in use: cache its device copy.
struct Cache { const void* key = nullptr; size_t n = 0; lodgs_gpu_scene* s = nullptr; };
}  // namespace

RenderOutput render(const LoDTree& tree, const Camera& cam, const FilterConfig& f,
                    const ShrinkMode& mode, const RenderOptions& opts) {
    static std::mutex mu;
    static Cache cache;
    std::lock_guard<std::mutex> lk(mu);
    if (cache.key != tree.mean_x.data() || cache.n != tree.node_count()) {
        if (cache.s) lodgs_gpu_scene_destroy(cache.s);
        const lodgs_tree_view v = view_of(tree);
        if (int rc = lodgs_gpu_scene_create(&v, 0, &cache.s)) rethrow(rc);
        cache = {tree.mean_x.data(), tree.node_count(), cache.s};
    }
    const lodgs_camera c = cam_of(cam);
    const lodgs_render_params p{
        f.tau_r, mode.tau, int32_t(mode.kind),
        LODGS_RENDER_STAGE_TIMING |
            (opts.collect_kpc ? LODGS_RENDER_KEEP_PAIRS | LODGS_RENDER_COLLECT_KPC : 0u) |
            (opts.filter_mode == FilterMode::serial ? LODGS_RENDER_FILTER_SERIAL : 0u)};
    RenderOutput out;
    out.image = Image::black(int(cam.width), int(cam.height));
    lodgs_render_stats st{};
    if (int rc = lodgs_gpu_render(cache.s, &c, &p, out.image.rgb.data(), &st)) rethrow(rc);
    out.stats.n_selected = st.n_selected;
    out.stats.n_pairs = st.n_pairs;
    out.stats.filter_passes = st.filter_passes;
    out.stats.filter_barriers = st.filter_barriers;
    out.stats.t_calc_ms = st.t_calc_ms;  // device stage times (LODGS_RENDER_STAGE_TIMING)
    out.stats.t_sync_ms = st.t_sync_ms;
    out.stats.t_prepr_ms = st.t_prepr_ms;
    out.stats.t_sort_ms = st.t_sort_ms;
    out.stats.t_alpha_ms = st.t_alpha_ms;
    if (opts.collect_kpc) {
        out.pairs.resize(st.n_pairs);
        out.kpc.resize(st.n_pairs);
        uint64_t n = 0;
        lodgs_gpu_read_pairs(cache.s, reinterpret_cast<lodgs_tile_pair*>(out.pairs.data()),
                             out.pairs.size(), &n);  // TilePair and lodgs_tile_pair share layout
        lodgs_gpu_read_kpc(cache.s, out.kpc.data(), out.kpc.size(), &n);
        BlendList& g = out.gaussians;  // RenderOutput::gaussians (rasterizer.hpp:93)
        const uint64_t ng = st.n_gaussians;
        for (auto* v : {&g.mean_x, &g.mean_y, &g.conic_a, &g.conic_b, &g.conic_c, &g.opacity,
                        &g.col_r, &g.col_g, &g.col_b, &g.radius})
            v->resize(ng);
        g.depth.resize(ng);
        g.node.resize(ng);
        lodgs_blend_list bl{ng,               g.mean_x.data(),  g.mean_y.data(),
                            g.conic_a.data(), g.conic_b.data(), g.conic_c.data(),
                            g.opacity.data(), g.col_r.data(),   g.col_g.data(),
                            g.col_b.data(),   g.radius.data(),  g.depth.data(),
                            g.node.data()};
        if (int rc = lodgs_gpu_read_gaussians(cache.s, &bl, ng)) rethrow(rc);
    }
    return out;
}
}  // namespace lodgs
