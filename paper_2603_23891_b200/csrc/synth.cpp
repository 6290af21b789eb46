// synth.cpp -- benchmark INPUT generation, kept out of the renderer library:
// the reference's synthetic scene generator + LoD builder (tree_builder.cpp:75-174,
// rng.hpp:11-33) and camera-path sampling (camera_path.cpp:18-180), restated in C++
// bit for bit (tests/test_oracle_cpu.py compares both with the compiled reference).
// SURVEY.md section 2 marks tree_builder / camera_path out of the hot path, so they
// build into _lib/liblodgs_synth.so (include/lodgs_synth.h), not liblodgs_b200.so.
// Compiled with -ffp-contract=off so every double expression rounds like the
// reference build (proj/CMakeLists.txt:13).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/lodgs_synth.h"
#include "host_util.h"

namespace fgs {

namespace {

using Quat = std::array<double, 4>;

// camera_path.cpp:23-50: rotation matrix -> quaternion (Shepperd branches).
Quat quat_from_rotation(const double* m) {
    const double trace = m[0] + m[4] + m[8];
    double w, x, y, z;
    if (trace > 0.0) {
        const double s = std::sqrt(trace + 1.0) * 2.0;
        w = 0.25 * s;
        x = (m[7] - m[5]) / s;
        y = (m[2] - m[6]) / s;
        z = (m[3] - m[1]) / s;
    } else if (m[0] > m[4] && m[0] > m[8]) {
        const double s = std::sqrt(1.0 + m[0] - m[4] - m[8]) * 2.0;
        w = (m[7] - m[5]) / s;
        x = 0.25 * s;
        y = (m[1] + m[3]) / s;
        z = (m[2] + m[6]) / s;
    } else if (m[4] > m[8]) {
        const double s = std::sqrt(1.0 + m[4] - m[0] - m[8]) * 2.0;
        w = (m[2] - m[6]) / s;
        x = (m[1] + m[3]) / s;
        y = 0.25 * s;
        z = (m[5] + m[7]) / s;
    } else {
        const double s = std::sqrt(1.0 + m[8] - m[0] - m[4]) * 2.0;
        w = (m[3] - m[1]) / s;
        x = (m[2] + m[6]) / s;
        y = (m[5] + m[7]) / s;
        z = 0.25 * s;
    }
    return {w, x, y, z};
}

// camera_path.cpp:52-75
Quat slerp(Quat a, Quat b, double t) {
    double d = a[0] * b[0] + a[1] * b[1] + a[2] * b[2] + a[3] * b[3];
    if (d < 0.0) {
        for (double& v : b) v = -v;
        d = -d;
    }
    double ka, kb;
    if (d > 0.9995) {
        ka = 1.0 - t;
        kb = t;
    } else {
        const double th = std::acos(std::clamp(d, -1.0, 1.0));
        const double sth = std::sin(th);
        ka = std::sin((1.0 - t) * th) / sth;
        kb = std::sin(t * th) / sth;
    }
    Quat q = {ka * a[0] + kb * b[0], ka * a[1] + kb * b[1], ka * a[2] + kb * b[2],
              ka * a[3] + kb * b[3]};
    const double n = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    for (double& v : q) v /= n;
    return q;
}

// core.hpp:70-85 rotation_matrix(w,x,y,z): normalises first.
void rotation_matrix(double w, double x, double y, double z, double* r) {
    const double n = std::sqrt(w * w + x * x + y * y + z * z);
    w /= n;
    x /= n;
    y /= n;
    z /= n;
    r[0] = 1 - 2 * (y * y + z * z);
    r[1] = 2 * (x * y - w * z);
    r[2] = 2 * (x * z + w * y);
    r[3] = 2 * (x * y + w * z);
    r[4] = 1 - 2 * (x * x + z * z);
    r[5] = 2 * (y * z - w * x);
    r[6] = 2 * (x * z - w * y);
    r[7] = 2 * (y * z + w * x);
    r[8] = 1 - 2 * (x * x + y * y);
}

}  // namespace

// camera_path.cpp:159-180
lodgs_camera interpolate(const lodgs_camera& a, const lodgs_camera& b, double t) {
    const double u = 1.0 - t;
    lodgs_camera c{};
    c.width = a.width;
    c.height = a.height;
    c.fx = u * a.fx + t * b.fx;
    c.fy = u * a.fy + t * b.fy;
    c.cx = u * a.cx + t * b.cx;
    c.cy = u * a.cy + t * b.cy;
    c.znear = u * a.znear + t * b.znear;
    c.zfar = u * a.zfar + t * b.zfar;
    for (int i = 0; i < 3; ++i)
        c.translation[i] = u * a.translation[i] + t * b.translation[i];
    const Quat q = slerp(quat_from_rotation(a.rotation), quat_from_rotation(b.rotation), t);
    rotation_matrix(q[0], q[1], q[2], q[3], c.rotation);
    return c;
}

// camera_path.cpp:126-157 (frame_count, sample, require_valid(path))
std::vector<lodgs_camera> sample_path(const lodgs_camera* keys, uint32_t n_keys,
                                      const uint32_t* samples) {
    if (n_keys == 0) throw Error(LODGS_ERR_VALIDATION, "camera path: at least one keyframe");
    for (uint32_t s = 0; s + 1 < n_keys; ++s)
        if (samples[s] < 1) throw Error(LODGS_ERR_VALIDATION, "camera path: sample counts >= 1");
    for (uint32_t k = 0; k < n_keys; ++k) {
        const auto v = validate_camera(keys[k]);
        if (!v.empty()) throw Error(LODGS_ERR_VALIDATION, join_violations("invalid camera", v, v.size()));
        if (keys[k].width != keys[0].width || keys[k].height != keys[0].height)
            throw Error(LODGS_ERR_VALIDATION,
                        "camera path: all keyframes share one image size");
    }
    std::vector<lodgs_camera> frames;
    for (uint32_t s = 0; s + 1 < n_keys; ++s)
        for (uint32_t k = 0; k < samples[s]; ++k)
            frames.push_back(interpolate(keys[s], keys[s + 1], double(k) / double(samples[s])));
    frames.push_back(keys[n_keys - 1]);
    return frames;
}

// ------------------------------------------------------ synthetic scenes --
namespace {

// rng.hpp:11-33 on std::mt19937_64, whose output the C++ standard pins.
struct Rng {
    std::mt19937_64 gen;
    explicit Rng(uint64_t seed) : gen(seed) {}
    double next_double() { return double(gen() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }
    uint64_t next_below(uint64_t n) { return gen() % n; }
};

uint64_t mix_seed(uint64_t seed, uint64_t item) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (item + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct Node {
    float mean[3], scale[3], quat[4], opacity, color[3];
};

const float kPalette[4][3] = {{0.9f, 0.2f, 0.2f}, {0.2f, 0.9f, 0.2f}, {0.2f, 0.2f, 0.9f},
                              {0.9f, 0.9f, 0.2f}};

}  // namespace

// tree_builder.cpp:126-174 generate_synthetic_scene + :94-124 build_tree.
uint64_t build_synthetic(const lodgs_synthetic_spec& s, const lodgs_build_config& c,
                         lodgs_tree_buffers* out, uint32_t* n_levels) {
    if (s.nx < 1 || s.ny < 1) throw Error(LODGS_ERR_VALIDATION, "scene spec: nx, ny >= 1");
    if (!(s.spacing > 0)) throw Error(LODGS_ERR_VALIDATION, "scene spec: spacing > 0");
    if (!(s.scale_min > 0 && s.scale_min <= s.scale_max))
        throw Error(LODGS_ERR_VALIDATION, "scene spec: 0 < scale_min <= scale_max");
    if (!(s.opacity_min > 0 && s.opacity_min <= s.opacity_max && s.opacity_max <= 1))
        throw Error(LODGS_ERR_VALIDATION, "scene spec: opacity range within (0,1]");
    if (s.congestion < 1) throw Error(LODGS_ERR_VALIDATION, "scene spec: congestion >= 1");
    if (c.depth < 1) throw Error(LODGS_ERR_VALIDATION, "build config: depth >= 1");
    if (!(c.shrink_factor > 0.0f && c.shrink_factor <= 0.8f))
        throw Error(LODGS_ERR_VALIDATION, "build config: shrink_factor in (0, 0.8]");
    if (c.children_per_node < 1 || c.children_per_node > 8)
        throw Error(LODGS_ERR_VALIDATION, "build config: children_per_node in {1..8}");

    const uint64_t n_roots = uint64_t(s.nx) * s.ny * s.congestion;
    const uint64_t cap = uint64_t(kRootParent);
    uint64_t total = 0, per_level = n_roots;
    for (uint32_t l = 0; l <= c.depth; ++l) {
        total += per_level;
        if (total >= cap) throw Error(LODGS_ERR_VALIDATION, "tree node count overflows index type");
        if (l < c.depth && per_level > cap / c.children_per_node)
            throw Error(LODGS_ERR_VALIDATION, "tree node count overflows index type");
        per_level *= c.children_per_node;
    }
    if (n_levels) *n_levels = c.depth + 1;
    if (!out) return total;

    auto put = [&](uint64_t i, const Node& n, uint32_t parent, bool leaf) {
        out->mean_x[i] = n.mean[0];
        out->mean_y[i] = n.mean[1];
        out->mean_z[i] = n.mean[2];
        out->scale_x[i] = n.scale[0];
        out->scale_y[i] = n.scale[1];
        out->scale_z[i] = n.scale[2];
        out->quat_w[i] = n.quat[0];
        out->quat_x[i] = n.quat[1];
        out->quat_y[i] = n.quat[2];
        out->quat_z[i] = n.quat[3];
        out->opacity[i] = n.opacity;
        out->color_r[i] = n.color[0];
        out->color_g[i] = n.color[1];
        out->color_b[i] = n.color[2];
        out->parent[i] = parent;
        out->leaf[i] = leaf ? 1 : 0;
    };

    // Roots: jittered grid, one stream per cell (tree_builder.cpp:142-172).
    const double spacing = s.spacing;
    const double x0 = -0.5 * spacing * (s.nx - 1);
    const double y0 = -0.5 * spacing * (s.ny - 1);
    uint64_t k = 0;
    for (uint32_t iy = 0; iy < s.ny; ++iy)
        for (uint32_t ix = 0; ix < s.nx; ++ix) {
            Rng rng(mix_seed(s.seed, uint64_t(iy) * s.nx + ix));
            for (uint32_t cc = 0; cc < s.congestion; ++cc) {
                Node n;
                n.mean[0] = float(x0 + ix * spacing + rng.uniform(-0.35, 0.35) * spacing);
                n.mean[1] = float(y0 + iy * spacing + rng.uniform(-0.35, 0.35) * spacing);
                n.mean[2] = float(rng.uniform(-0.5, 0.5) * spacing);
                n.scale[0] = float(rng.uniform(s.scale_min, s.scale_max));
                n.scale[1] = float(rng.uniform(s.scale_min, s.scale_max));
                n.scale[2] = float(rng.uniform(s.scale_min, s.scale_max));
                const double u1 = rng.next_double();
                const double a = 2.0 * 3.141592653589793 * rng.next_double();
                const double b = 2.0 * 3.141592653589793 * rng.next_double();
                const double r1 = std::sqrt(1.0 - u1), r2 = std::sqrt(u1);
                n.quat[0] = float(r2 * std::cos(b));
                n.quat[1] = float(r1 * std::sin(a));
                n.quat[2] = float(r1 * std::cos(a));
                n.quat[3] = float(r2 * std::sin(b));
                n.opacity = float(rng.uniform(s.opacity_min, s.opacity_max));
                const uint64_t pi = rng.next_below(4);
                for (int ch = 0; ch < 3; ++ch) n.color[ch] = kPalette[pi][ch];
                put(k++, n, kRootParent, false);  // build_tree clears leaf on roots
            }
        }
    out->level_offsets[0] = 0;

    // Levels: corner-offset children (tree_builder.cpp:94-124).
    uint64_t begin = 0, end = k;
    for (uint32_t level = 1; level <= c.depth; ++level) {
        out->level_offsets[level] = uint32_t(k);
        const bool leaf = level == c.depth;
        for (uint64_t p = begin; p < end; ++p) {
            double rot[9];
            rotation_matrix(out->quat_w[p], out->quat_x[p], out->quat_y[p], out->quat_z[p], rot);
            const double mean[3] = {out->mean_x[p], out->mean_y[p], out->mean_z[p]};
            const float sx = out->scale_x[p], sy = out->scale_y[p], sz = out->scale_z[p];
            uint32_t corners[8];
            for (uint32_t i = 0; i < 8; ++i) corners[i] = i;
            if (c.children_per_node != 8) {
                Rng rng(mix_seed(c.seed, p));
                for (uint32_t i = 0; i < c.children_per_node; ++i) {
                    const uint32_t j = i + uint32_t(rng.next_below(8 - i));
                    std::swap(corners[i], corners[j]);
                }
                for (uint32_t a = 1; a < c.children_per_node; ++a)  // sort the chosen corners
                    for (uint32_t b2 = a; b2 > 0 && corners[b2 - 1] > corners[b2]; --b2)
                        std::swap(corners[b2 - 1], corners[b2]);
            }
            for (uint32_t ci = 0; ci < c.children_per_node; ++ci) {
                const uint32_t cn = corners[ci];
                const double off[3] = {(cn & 1 ? 0.5 : -0.5) * double(sx),
                                       (cn & 2 ? 0.5 : -0.5) * double(sy),
                                       (cn & 4 ? 0.5 : -0.5) * double(sz)};
                const double rv[3] = {rot[0] * off[0] + rot[1] * off[1] + rot[2] * off[2],
                                      rot[3] * off[0] + rot[4] * off[1] + rot[5] * off[2],
                                      rot[6] * off[0] + rot[7] * off[1] + rot[8] * off[2]};
                Node n;
                n.mean[0] = float(mean[0] + rv[0]);
                n.mean[1] = float(mean[1] + rv[1]);
                n.mean[2] = float(mean[2] + rv[2]);
                n.scale[0] = sx * c.shrink_factor;
                n.scale[1] = sy * c.shrink_factor;
                n.scale[2] = sz * c.shrink_factor;
                n.quat[0] = out->quat_w[p];
                n.quat[1] = out->quat_x[p];
                n.quat[2] = out->quat_y[p];
                n.quat[3] = out->quat_z[p];
                n.opacity = out->opacity[p];
                n.color[0] = out->color_r[p];
                n.color[1] = out->color_g[p];
                n.color[2] = out->color_b[p];
                put(k++, n, uint32_t(p), leaf);
            }
        }
        begin = end;
        end = k;
    }
    return k;
}

}  // namespace fgs

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
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return LODGS_ERR_INTERNAL;
    }
}

void need(const void* p, const char* what) {
    if (!p) throw fgs::Error(LODGS_ERR_VALIDATION, std::string("null argument: ") + what);
}
}  // namespace

extern "C" {

const char* lodgs_synth_last_error(void) { return g_last_error.c_str(); }

int lodgs_camera_path_sample(const lodgs_camera* keyframes, uint32_t n_keyframes,
                             const uint32_t* samples, lodgs_camera* out, uint64_t out_cap,
                             uint64_t* n_frames) {
    return guarded([&] {
        need(keyframes, "keyframes");
        if (n_keyframes > 1) need(samples, "samples");
        const auto f = fgs::sample_path(keyframes, n_keyframes, samples);
        if (n_frames) *n_frames = f.size();
        if (out) {
            if (out_cap < f.size()) throw fgs::Error(LODGS_ERR_VALIDATION, "camera path: capacity");
            std::memcpy(out, f.data(), f.size() * sizeof(lodgs_camera));
        }
    });
}

int lodgs_build_synthetic_tree(const lodgs_synthetic_spec* spec, const lodgs_build_config* cfg,
                               lodgs_tree_buffers* out, uint64_t* n_nodes, uint32_t* n_levels) {
    return guarded([&] {
        need(spec, "spec");
        need(cfg, "cfg");
        const uint64_t n = fgs::build_synthetic(*spec, *cfg, out, n_levels);
        if (n_nodes) *n_nodes = n;
    });
}

}  // extern "C"
