// capi.cpp -- extern "C" boundary (include/lodgs_gpu.h).  Every entry point
// converts C++ exceptions into lodgs_status codes + a thread-local message,
// mirroring how the reference CLI maps ValidationError / IoError to exit
// codes 2 / 3 (cli.cpp:392-408).
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "host_util.h"
#include "scene.h"

struct lodgs_gpu_scene {
    fgs::GpuScene* impl;
};

namespace {
thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return LODGS_OK;
    } catch (const fgs::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return LODGS_ERR_INTERNAL;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return LODGS_ERR_INTERNAL;
    }
}

void copy_msg(const std::string& s, char* msg, size_t cap) {
    if (!msg || cap == 0) return;
    const size_t k = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(msg, s.data(), k);
    msg[k] = 0;
}

fgs::GpuScene& S(lodgs_gpu_scene* s) {
    if (!s || !s->impl) throw fgs::Error(LODGS_ERR_VALIDATION, "null scene");
    return *s->impl;
}

void need(const void* p, const char* what) {
    if (!p) throw fgs::Error(LODGS_ERR_VALIDATION, std::string("null argument: ") + what);
}
}  // namespace

extern "C" {

const char* lodgs_gpu_last_error(void) { return g_last_error.c_str(); }
int lodgs_gpu_abi_version(void) { return LODGS_GPU_ABI_VERSION; }

int lodgs_gpu_device_count(int* count) {
    return guarded([&] {
        need(count, "count");
        *count = 0;
        const cudaError_t e = cudaGetDeviceCount(count);
        if (e != cudaSuccess) {
            *count = 0;
            cudaGetLastError();
            throw fgs::Error(LODGS_ERR_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
        }
    });
}

int lodgs_validate_tree(const lodgs_tree_view* tree, uint64_t* n_violations, char* msg,
                        size_t msg_cap) {
    return guarded([&] {
        need(tree, "tree");
        uint64_t nv = 0;
        const auto v = fgs::validate_tree(*tree, &nv);
        if (n_violations) *n_violations = nv;
        copy_msg(nv ? fgs::join_violations("invalid tree", v, nv) : std::string(), msg, msg_cap);
    });
}

int lodgs_validate_camera(const lodgs_camera* cam, uint64_t* n_violations, char* msg,
                          size_t msg_cap) {
    return guarded([&] {
        need(cam, "cam");
        const auto v = fgs::validate_camera(*cam);
        if (n_violations) *n_violations = v.size();
        copy_msg(v.empty() ? std::string() : fgs::join_violations("invalid camera", v, v.size()),
                 msg, msg_cap);
    });
}

int lodgs_camera_geom(const lodgs_camera* cam, double out44[44]) {
    return guarded([&] {
        need(cam, "cam");
        need(out44, "out44");
        const fgs::Geom g = fgs::camera_geom(*cam);
        static_assert(sizeof(fgs::Geom) == 44 * sizeof(double), "CameraGeom is 44 doubles");
        std::memcpy(out44, &g, sizeof g);
    });
}

int lodgs_gpu_scene_create(const lodgs_tree_view* tree, int device, lodgs_gpu_scene** out) {
    return guarded([&] {
        need(tree, "tree");
        need(out, "out");
        *out = nullptr;
        auto* impl = new fgs::GpuScene(*tree, device);
        *out = new lodgs_gpu_scene{impl};
    });
}

int lodgs_gpu_scene_load(const char* path, int device, lodgs_gpu_scene** out,
                         double* timing_ms) {
    return guarded([&] {
        need(path, "path");
        need(out, "out");
        *out = nullptr;
        auto* impl = new fgs::GpuScene(std::string(path), device, timing_ms);
        *out = new lodgs_gpu_scene{impl};
    });
}

int lodgs_gpu_scene_info(lodgs_gpu_scene* scene, uint64_t* n_nodes, uint32_t* n_levels,
                         uint32_t* level_offsets, uint32_t cap, float* shrink_factor) {
    return guarded([&] {
        const auto& s = S(scene);
        if (n_nodes) *n_nodes = s.n_nodes();
        if (n_levels) *n_levels = uint32_t(s.n_levels());
        if (shrink_factor) *shrink_factor = s.shrink_factor();
        if (level_offsets) {
            if (cap < uint32_t(s.n_levels()))
                throw fgs::Error(LODGS_ERR_VALIDATION, "scene_info: capacity too small");
            for (int l = 0; l < s.n_levels(); ++l)
                level_offsets[l] = uint32_t(s.level_begin()[size_t(l)]);
        }
    });
}

int lodgs_gpu_scene_destroy(lodgs_gpu_scene* scene) {
    return guarded([&] {
        if (!scene) return;
        delete scene->impl;
        delete scene;
    });
}

int lodgs_gpu_scene_stream(lodgs_gpu_scene* scene, void** stream) {
    return guarded([&] {
        need(stream, "stream");
        *stream = static_cast<void*>(S(scene).stream());
    });
}

int lodgs_gpu_scene_reserve(lodgs_gpu_scene* scene, uint64_t max_pairs) {
    return guarded([&] { S(scene).reserve_pairs(max_pairs); });
}

int lodgs_gpu_scene_memory(lodgs_gpu_scene* scene, uint64_t* bytes) {
    return guarded([&] {
        need(bytes, "bytes");
        *bytes = S(scene).device_bytes();
    });
}

int lodgs_gpu_render(lodgs_gpu_scene* scene, const lodgs_camera* cam,
                     const lodgs_render_params* params, float* image_host,
                     lodgs_render_stats* stats) {
    return guarded([&] {
        need(cam, "cam");
        need(params, "params");
        S(scene).render(*cam, *params, image_host, stats);
    });
}

int lodgs_gpu_render_batch(lodgs_gpu_scene* scene, const lodgs_camera* cams, uint64_t n,
                           const lodgs_render_params* params, float* const* images_host,
                           lodgs_render_stats* stats) {
    return guarded([&] {
        if (n) need(cams, "cams");
        need(params, "params");
        S(scene).render_batch(cams, n, *params, images_host, stats);
    });
}

int lodgs_gpu_render_views_async(lodgs_gpu_scene* scene, const lodgs_camera* cams, uint64_t n,
                                 const lodgs_render_params* params, float* const* images_host) {
    return guarded([&] {
        if (n) need(cams, "cams");
        need(params, "params");
        S(scene).enqueue_views_async(cams, n, *params, images_host);
    });
}

int lodgs_gpu_render_async(lodgs_gpu_scene* scene, const lodgs_camera* cam,
                           const lodgs_render_params* params, float* image_host) {
    return guarded([&] {
        need(cam, "cam");
        need(params, "params");
        S(scene).enqueue_async(*cam, *params, image_host);
    });
}

int lodgs_gpu_sync(lodgs_gpu_scene* scene, lodgs_render_stats* stats) {
    return guarded([&] { S(scene).sync_async(stats); });
}

int lodgs_gpu_take_totals(lodgs_gpu_scene* scene, uint64_t* frames, uint64_t* sum_selected,
                          uint64_t* sum_pairs, uint64_t* sum_sort_bytes) {
    return guarded(
        [&] { S(scene).take_totals(frames, sum_selected, sum_pairs, sum_sort_bytes); });
}


int lodgs_gpu_scene_set_inflight(lodgs_gpu_scene* scene, int frames) {
    return guarded([&] { S(scene).set_inflight(frames); });
}

int lodgs_gpu_scene_set_sh(lodgs_gpu_scene* scene, int degree, const float* sh_rest,
                           uint64_t n_nodes) {
    return guarded([&] { S(scene).set_sh(degree, sh_rest, n_nodes); });
}

int lodgs_gpu_join(lodgs_gpu_scene* scene) {
    return guarded([&] { S(scene).join(); });
}

int lodgs_gpu_profile(lodgs_gpu_scene* scene, int enable) {
    return guarded([&] { S(scene).profile(enable != 0); });
}

int lodgs_gpu_profile_read(lodgs_gpu_scene* scene, uint64_t* frames, double stage_ms[6]) {
    return guarded([&] {
        need(stage_ms, "stage_ms");
        const uint64_t f = S(scene).profile_read(stage_ms);
        if (frames) *frames = f;
    });
}

int lodgs_gpu_read_image(lodgs_gpu_scene* scene, float* out) {
    return guarded([&] {
        need(out, "out");
        S(scene).read_image(out);
    });
}

int lodgs_gpu_image_device_ptr(lodgs_gpu_scene* scene, const float** dev_ptr) {
    return guarded([&] {
        need(dev_ptr, "dev_ptr");
        *dev_ptr = S(scene).image_device();
    });
}

int lodgs_gpu_read_selected(lodgs_gpu_scene* scene, uint32_t* out, uint64_t cap, uint64_t* n) {
    return guarded([&] {
        const uint64_t k = S(scene).read_selected(out, cap);
        if (n) *n = k;
    });
}

int lodgs_gpu_read_pairs(lodgs_gpu_scene* scene, lodgs_tile_pair* out, uint64_t cap,
                         uint64_t* n) {
    return guarded([&] {
        const uint64_t k = S(scene).read_pairs(out, cap);
        if (n) *n = k;
    });
}

int lodgs_gpu_read_gaussians(lodgs_gpu_scene* scene, lodgs_blend_list* out, uint64_t cap) {
    return guarded([&] {
        need(out, "out");
        S(scene).read_gaussians(out, cap);
    });
}

int lodgs_gpu_read_kpc(lodgs_gpu_scene* scene, double* out, uint64_t cap, uint64_t* n) {
    return guarded([&] {
        const uint64_t k = S(scene).read_kpc(out, cap);
        if (n) *n = k;
    });
}

int lodgs_gpu_calibrate(lodgs_gpu_scene* scene, const lodgs_camera* views, uint32_t n_views,
                        double lambda_g, double tau_r, lodgs_calibration* out, double* per_view) {
    return guarded([&] {
        need(out, "out");
        if (n_views) need(views, "views");
        if (!(tau_r > 0)) throw fgs::Error(LODGS_ERR_VALIDATION, "filter config: tau_r > 0");
        S(scene).calibrate(views, n_views, lambda_g, tau_r, out, per_view);
    });
}

int lodgs_gpu_read_counts(lodgs_gpu_scene* scene, uint32_t* per_gaussian, uint64_t cap_g,
                          uint32_t* per_tile, uint64_t cap_t) {
    return guarded([&] { S(scene).read_counts(per_gaussian, cap_g, per_tile, cap_t); });
}

int lodgs_gpu_filter(lodgs_gpu_scene* scene, const lodgs_camera* cam, double tau_r,
                     uint32_t* selected, uint64_t cap, uint64_t* n_selected, int32_t* passes,
                     int32_t* barriers) {
    return guarded([&] {
        need(cam, "cam");
        std::vector<uint32_t> sel;
        const uint64_t ns = S(scene).filter(*cam, tau_r, sel);
        if (n_selected) *n_selected = ns;
        if (passes) *passes = 2;
        if (barriers) *barriers = 2;
        if (selected) {
            if (cap < ns) throw fgs::Error(LODGS_ERR_VALIDATION, "filter: capacity too small");
            std::memcpy(selected, sel.data(), ns * 4);
        }
    });
}

int lodgs_gpu_filter_serial(lodgs_gpu_scene* scene, const lodgs_camera* cam, double tau_r,
                            uint32_t* selected, uint64_t cap, uint64_t* n_selected,
                            int32_t* passes, int32_t* barriers, double* level_ms) {
    return guarded([&] {
        need(cam, "cam");
        std::vector<uint32_t> sel;
        int32_t ps = 0;
        const uint64_t ns = S(scene).filter_serial(*cam, tau_r, sel, &ps, level_ms);
        if (n_selected) *n_selected = ns;
        if (passes) *passes = ps;
        if (barriers) *barriers = ps;
        if (selected) {
            if (cap < ns) throw fgs::Error(LODGS_ERR_VALIDATION, "filter: capacity too small");
            std::memcpy(selected, sel.data(), ns * 4);
        }
    });
}

int lodgs_gpu_read_image_rgb8(lodgs_gpu_scene* scene, uint8_t* out) {
    return guarded([&] {
        need(out, "out");
        S(scene).read_image_rgb8(out);
    });
}

int lodgs_gpu_set_reference_image(lodgs_gpu_scene* scene) {
    return guarded([&] { S(scene).set_reference_image(); });
}

int lodgs_gpu_compare_reference(lodgs_gpu_scene* scene, double* psnr, double* ssim) {
    return guarded([&] { S(scene).compare_reference(psnr, ssim); });
}

int lodgs_gpu_image_metrics(const float* a, const float* b, int width, int height, double* psnr,
                            double* ssim) {
    return guarded([&] {
        need(a, "a");
        need(b, "b");
        fgs::stage_image_metrics(a, b, width, height, psnr, ssim);
    });
}

int lodgs_gpu_mark(lodgs_gpu_scene* scene, const lodgs_camera* cam, uint64_t begin, uint64_t end,
                   double tau_r, uint8_t* vis, uint8_t* qpass, double* radius) {
    return guarded([&] {
        need(cam, "cam");
        need(vis, "vis");
        need(qpass, "qpass");
        S(scene).mark(*cam, begin, end, tau_r, vis, qpass, radius);
    });
}

int lodgs_gpu_prepare(lodgs_gpu_scene* scene, const lodgs_camera* cam, const uint32_t* selected,
                      uint64_t n_sel, int32_t shrink_kind, double tau, lodgs_blend_list* out) {
    return guarded([&] {
        need(cam, "cam");
        need(out, "out");
        if (n_sel) need(selected, "selected");
        if (shrink_kind < 0 || shrink_kind > 2)
            throw fgs::Error(LODGS_ERR_VALIDATION, "shrink mode: unknown kind");
        S(scene).prepare(*cam, selected, n_sel, shrink_kind, tau, out);
    });
}

int lodgs_gpu_bin_to_tiles(const lodgs_blend_list* list, int width, int height,
                           lodgs_tile_pair* out, uint64_t cap, uint64_t* n_pairs) {
    return guarded([&] {
        need(list, "list");
        uint64_t np = 0;
        fgs::stage_bin_to_tiles(*list, width, height, out, cap, &np);
        if (n_pairs) *n_pairs = np;
    });
}

int lodgs_gpu_sort_pairs(lodgs_tile_pair* pairs, uint64_t n) {
    return guarded([&] {
        if (n) need(pairs, "pairs");
        fgs::stage_sort_pairs(pairs, n);
    });
}

int lodgs_gpu_alpha_blend(const lodgs_tile_pair* sorted, uint64_t n, const lodgs_blend_list* list,
                          int width, int height, uint32_t flags, float* image) {
    return guarded([&] {
        need(list, "list");
        need(image, "image");
        if (n) need(sorted, "sorted");
        fgs::stage_alpha_blend(sorted, n, *list, width, height, flags, image);
    });
}

int lodgs_gpu_host_alloc(uint64_t bytes, void** ptr) {
    return guarded([&] {
        need(ptr, "ptr");
        FGS_CUDA(cudaMallocHost(ptr, bytes ? bytes : 1));
    });
}

int lodgs_gpu_host_free(void* ptr) {
    return guarded([&] {
        if (ptr) FGS_CUDA(cudaFreeHost(ptr));
    });
}

}  // extern "C"
