// shim_check.cpp -- the drop-in, linked and run.
//
// One binary holds the UNMODIFIED reference library (oracle/_ref objects, compiled
// from /root/reference's sources by oracle/Makefile) with its lodgs::render replaced
// by integration/rasterizer_b200.cpp -- the C++ shim INTEGRATION.md tells a
// maintainer to add -- over liblodgs_b200.so.  The reference's own render is kept
// under another name (objcopy --redefine-sym: render -> render_ref), and so are CPU
// copies of the reference code that calls render (run_bench -> run_bench_ref,
// calibrate -> calibrate_ref), so the same binary compares:
//
//   1. a production frame (render, B200) against the reference's render (CPU):
//      n_selected / n_pairs / passes / barriers equal, image max-abs <= 1e-3;
//   2. a collect_kpc frame: image, sorted pairs, kpc and BlendList bit-identical;
//   3. the reference's run_bench (bench.cpp:114-168) over filter x shrink combos,
//      with every render on the B200, against run_bench_ref on the CPU: every
//      FrameRow / AggregateRow field except the timings identical;
//   4. the reference's calibrate (metrics.cpp:94-108) on the B200 against the CPU.
//
// Prints one JSON object; tests/test_gpu_integration.py runs it on the GPU box.
// TEST INFRASTRUCTURE (links the reference): built into oracle/_ref only.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "lodgs/bench.hpp"
#include "lodgs/metrics.hpp"
#include "lodgs/rasterizer.hpp"
#include "lodgs/tree_builder.hpp"

namespace lodgs {
RenderOutput render_ref(const LoDTree& tree, const Camera& cam, const FilterConfig& filter,
                        const ShrinkMode& mode, const RenderOptions& opts);
BenchReport run_bench_ref(const LoDTree& tree, const std::vector<Camera>& frames,
                          const std::vector<BenchCombo>& combos, const FilterConfig& filter_cfg);
CalibrationReport calibrate_ref(const LoDTree& tree, const std::vector<Camera>& views,
                                double lambda_g, const FilterConfig& filter);
}  // namespace lodgs

using namespace lodgs;

namespace {
double max_abs(const Image& a, const Image& b) {
    double m = 0;
    for (size_t i = 0; i < a.rgb.size(); ++i) m = std::max(m, double(std::fabs(a.rgb[i] - b.rgb[i])));
    return m;
}
bool same_bytes(const void* a, const void* b, size_t n) { return n == 0 || std::memcmp(a, b, n) == 0; }
template <class V>
bool same_vec(const V& a, const V& b) {
    return a.size() == b.size() && same_bytes(a.data(), b.data(), a.size() * sizeof(a[0]));
}
Camera front(uint32_t w, uint32_t h, double f, double tx, double ty, double tz) {
    Camera c;
    c.width = w;
    c.height = h;
    c.fx = c.fy = f;
    c.cx = w / 2.0;
    c.cy = h / 2.0;
    c.world_to_cam_translation = {tx, ty, tz};
    return c;
}
}  // namespace

int main() {
    // cfg 1: 37x37 roots, L = 2, seeds 1 / 7
    SyntheticSceneSpec spec;
    spec.nx = spec.ny = 37;
    spec.seed = 1;
    TreeBuildConfig bc;
    bc.depth = 2;
    bc.seed = 7;
    const LoDTree tree = build_tree(generate_synthetic_scene(spec), bc);
    FilterConfig fc;
    fc.tau_r = 3.0;
    fc.worker_count = std::max(1u, std::thread::hardware_concurrency());
    const Camera cam = front(800, 600, 100.0, 0.0, 0.0, 12.0);
    RenderOptions ro;
    ro.worker_count = fc.worker_count;

    // 1. production frame
    const RenderOutput g = render(tree, cam, fc, ShrinkMode::three_sigma(), ro);
    const RenderOutput r = render_ref(tree, cam, fc, ShrinkMode::three_sigma(), ro);
    const double err = max_abs(g.image, r.image);
    const bool fast_ok = g.stats.n_selected == r.stats.n_selected &&
                         g.stats.n_pairs == r.stats.n_pairs &&
                         g.stats.filter_passes == r.stats.filter_passes &&
                         g.stats.filter_barriers == r.stats.filter_barriers && err <= 1e-3 &&
                         psnr(g.image, r.image) > 60.0;

    // 2. collect_kpc frame: everything bit-identical
    RenderOptions rk = ro;
    rk.collect_kpc = true;
    const RenderOutput gk = render(tree, cam, fc, ShrinkMode::three_sigma(), rk);
    const RenderOutput rkf = render_ref(tree, cam, fc, ShrinkMode::three_sigma(), rk);
    const BlendList& a = gk.gaussians;
    const BlendList& b = rkf.gaussians;
    const bool kpc_ok = same_vec(gk.image.rgb, rkf.image.rgb) && gk.pairs.size() == rkf.pairs.size() &&
                        same_bytes(gk.pairs.data(), rkf.pairs.data(), gk.pairs.size() * sizeof(TilePair)) &&
                        same_vec(gk.kpc, rkf.kpc) && same_vec(a.mean_x, b.mean_x) &&
                        same_vec(a.mean_y, b.mean_y) && same_vec(a.conic_a, b.conic_a) &&
                        same_vec(a.conic_b, b.conic_b) && same_vec(a.conic_c, b.conic_c) &&
                        same_vec(a.opacity, b.opacity) && same_vec(a.col_r, b.col_r) &&
                        same_vec(a.col_g, b.col_g) && same_vec(a.col_b, b.col_b) &&
                        same_vec(a.radius, b.radius) && same_vec(a.depth, b.depth) &&
                        same_vec(a.node, b.node);

    // 4. calibrate (instrumented three-sigma renders) on the B200 vs the CPU
    std::vector<Camera> views;
    for (int i = 0; i < 3; ++i) views.push_back(front(800, 600, 100.0, 0.7 * i, -0.4 * i, 12.0 + i));
    const CalibrationReport cg = calibrate(tree, views, 0.2, fc);
    const CalibrationReport cr = calibrate_ref(tree, views, 0.2, fc);
    const bool calib_ok = cg.per_view == cr.per_view && cg.scene_mean == cr.scene_mean && cg.n_views == cr.n_views &&
                          cg.tau == cr.tau && cg.histogram.bins == cr.histogram.bins;

    // 3. the reference bench matrix: filter (parallel / serial) x shrink (3 sigma /
    //    fixed / adaptive at the calibrated tau), every render through the shim
    const std::vector<BenchCombo> combos = {
        {FilterMode::parallel, ShrinkMode::three_sigma()},
        {FilterMode::parallel, ShrinkMode::fixed()},
        {FilterMode::parallel, ShrinkMode::adaptive(cr.tau)},
        {FilterMode::serial, ShrinkMode::three_sigma()},
        {FilterMode::serial, ShrinkMode::adaptive(cr.tau)}};
    const BenchReport bg = run_bench(tree, views, combos, fc);
    const BenchReport br = run_bench_ref(tree, views, combos, fc);
    bool bench_ok = bg.frames.size() == br.frames.size() && bg.aggregates.size() == br.aggregates.size();
    for (size_t i = 0; bench_ok && i < bg.frames.size(); ++i) {
        const FrameRow &x = bg.frames[i], &y = br.frames[i];
        bench_ok = x.frame == y.frame && x.filter_mode == y.filter_mode &&
                   x.shrink_mode == y.shrink_mode && x.n_pairs == y.n_pairs &&
                   x.n_low == y.n_low && x.barriers == y.barriers;
    }
    double fps_g = 0, fps_r = 0;
    for (size_t i = 0; bench_ok && i < bg.aggregates.size(); ++i) {
        const AggregateRow &x = bg.aggregates[i], &y = br.aggregates[i];
        bench_ok = x.filter_mode == y.filter_mode && x.shrink_mode == y.shrink_mode &&
                   x.mean_pairs == y.mean_pairs && x.barriers == y.barriers &&
                   x.histogram.bins == y.histogram.bins &&
                   format_metric(x.psnr_vs_ref) == format_metric(y.psnr_vs_ref) &&
                   format_metric(x.ssim_vs_ref) == format_metric(y.ssim_vs_ref);
        if (i == 0) {
            fps_g = x.fps;
            fps_r = y.fps;
        }
    }

    std::printf(
        "{\"nodes\": %zu, \"n_selected\": %zu, \"n_pairs\": %llu, \"max_abs\": %.3g, "
        "\"fast_ok\": %s, \"kpc_ok\": %s, \"calib_ok\": %s, \"tau\": %.17g, \"bench_ok\": %s, "
        "\"bench_rows\": %zu, \"bench_fps_b200\": %.3f, \"bench_fps_reference\": %.3f, "
        "\"t_calc_ms\": %.4f, \"t_sync_ms\": %.4f, \"t_prepr_ms\": %.4f, \"t_sort_ms\": %.4f, "
        "\"t_alpha_ms\": %.4f}\n",
        tree.node_count(), g.stats.n_selected, (unsigned long long)g.stats.n_pairs, err,
        fast_ok ? "true" : "false", kpc_ok ? "true" : "false", calib_ok ? "true" : "false", cr.tau,
        bench_ok ? "true" : "false", bg.frames.size(), fps_g, fps_r, g.stats.t_calc_ms,
        g.stats.t_sync_ms, g.stats.t_prepr_ms, g.stats.t_sort_ms, g.stats.t_alpha_ms);
    std::fputs(bench_json(bg).c_str(), stderr);
    return (fast_ok && kpc_ok && calib_ok && bench_ok) ? 0 : 1;
}
