// host_util.cpp -- host-side scene utilities of the lodgs API, restated in
// C++ for the B200 build: tree / camera validation (scene.cpp:89-199),
// CameraGeom::make (projection.cpp:11-38), camera-path sampling
// (camera_path.cpp:18-180) and the synthetic scene generator + LoD builder
// used for benchmark inputs (tree_builder.cpp:75-174, rng.hpp:11-33).
// None of this is per-frame GPU work; it runs once per upload / per camera.
// Compiled with -ffp-contract=off so every double expression rounds like
// the reference build (proj/CMakeLists.txt:13).
#include "host_util.h"

#include <algorithm>
#include <cmath>
#include <random>
#include <sstream>

namespace fgs {

// ------------------------------------------------------------ validation --
bool validate_tree_header(const lodgs_tree_view& t, std::vector<std::string>& out,
                          uint64_t& count) {
    auto add = [&](const std::string& rule) {
        ++count;
        if (out.size() < 9) out.push_back("tree: " + rule);
    };
    const uint64_t n = t.n_nodes;
    const float* ptrs[] = {t.mean_x, t.mean_y, t.mean_z, t.scale_x, t.scale_y,
                           t.scale_z, t.quat_w, t.quat_x, t.quat_y, t.quat_z,
                           t.opacity, t.color_r, t.color_g, t.color_b};
    bool arrays_ok = true;
    for (const float* p : ptrs) arrays_ok = arrays_ok && (p != nullptr || n == 0);
    if (!arrays_ok || (n && (!t.parent || !t.leaf))) {
        add("field arrays equal length");
        return false;
    }
    if (!(t.shrink_factor > 0.0f && t.shrink_factor < 1.0f)) add("shrink_factor in (0,1)");
    auto level_end = [&](uint32_t l) -> uint64_t {
        return l + 1 < t.n_levels ? t.level_offsets[l + 1] : n;
    };
    bool offsets_ok = t.n_levels > 0 && t.level_offsets && t.level_offsets[0] == 0;
    for (uint32_t l = 0; offsets_ok && l < t.n_levels; ++l)
        offsets_ok = t.level_offsets[l] <= level_end(l) && level_end(l) <= n;
    if (n > 0 && !offsets_ok) {
        add("level_offsets monotone in [0, node_count]");
        return false;
    }
    if (n == 0) {
        if (t.n_levels != 0) add("level_offsets empty for empty tree");
        return false;
    }
    return true;
}

const char* node_rule_name(int k) {
    static const char* names[9] = {"all fields finite", "unit quaternion", "scale > 0",
                                   "opacity in (0,1]", "color in [0,1]", "level-0 parent is ROOT",
                                   "parent index in range", "parent level == level - 1",
                                   "leaf iff childless"};
    return (k >= 0 && k < 9) ? names[k] : "?";
}

std::vector<std::string> validate_tree(const lodgs_tree_view& t, uint64_t* n_violations) {
    std::vector<std::string> out;
    uint64_t count = 0;
    auto add = [&](int64_t node, const std::string& rule) {
        ++count;
        if (out.size() < 9) {
            if (node < 0)
                out.push_back("tree: " + rule);
            else
                out.push_back("node " + std::to_string(node) + ": " + rule);
        }
    };
    const uint64_t n = t.n_nodes;
    const float* ptrs[] = {t.mean_x, t.mean_y, t.mean_z, t.scale_x, t.scale_y,
                           t.scale_z, t.quat_w, t.quat_x, t.quat_y, t.quat_z,
                           t.opacity, t.color_r, t.color_g, t.color_b};
    bool arrays_ok = true;
    for (const float* p : ptrs) arrays_ok = arrays_ok && (p != nullptr || n == 0);
    if (!arrays_ok || (n && (!t.parent || !t.leaf))) {
        add(-1, "field arrays equal length");
        if (n_violations) *n_violations = count;
        return out;
    }
    if (!(t.shrink_factor > 0.0f && t.shrink_factor < 1.0f)) add(-1, "shrink_factor in (0,1)");
    auto level_end = [&](uint32_t l) -> uint64_t {
        return l + 1 < t.n_levels ? t.level_offsets[l + 1] : n;
    };
    bool offsets_ok = t.n_levels > 0 && t.level_offsets && t.level_offsets[0] == 0;
    for (uint32_t l = 0; offsets_ok && l < t.n_levels; ++l)
        offsets_ok = t.level_offsets[l] <= level_end(l) && level_end(l) <= n;
    if (n > 0 && !offsets_ok) {
        add(-1, "level_offsets monotone in [0, node_count]");
        if (n_violations) *n_violations = count;
        return out;
    }
    if (n == 0) {
        if (t.n_levels != 0) add(-1, "level_offsets empty for empty tree");
        if (n_violations) *n_violations = count;
        return out;
    }
    std::vector<uint32_t> level_of(n);
    for (uint32_t l = 0; l < t.n_levels; ++l)
        for (uint64_t i = t.level_offsets[l]; i < level_end(l); ++i) level_of[i] = l;
    std::vector<uint8_t> has_child(n, 0);
    for (uint64_t i = 0; i < n; ++i)
        if (t.parent[i] != kRootParent && t.parent[i] < n) has_child[t.parent[i]] = 1;
    auto fin = [](float v) { return std::isfinite(v); };
    for (uint64_t i = 0; i < n; ++i) {
        if (!fin(t.mean_x[i]) || !fin(t.mean_y[i]) || !fin(t.mean_z[i]) || !fin(t.scale_x[i]) ||
            !fin(t.scale_y[i]) || !fin(t.scale_z[i]) || !fin(t.quat_x[i]) || !fin(t.quat_y[i]) ||
            !fin(t.quat_z[i]) || !fin(t.quat_w[i]) || !fin(t.opacity[i]) || !fin(t.color_r[i]) ||
            !fin(t.color_g[i]) || !fin(t.color_b[i])) {
            add(int64_t(i), "all fields finite");
            continue;
        }
        const double qn = std::sqrt(double(t.quat_w[i]) * t.quat_w[i] + double(t.quat_x[i]) * t.quat_x[i] +
                                    double(t.quat_y[i]) * t.quat_y[i] + double(t.quat_z[i]) * t.quat_z[i]);
        if (std::abs(qn - 1.0) > 1e-6) add(int64_t(i), "unit quaternion");
        if (!(t.scale_x[i] > 0 && t.scale_y[i] > 0 && t.scale_z[i] > 0)) add(int64_t(i), "scale > 0");
        if (!(t.opacity[i] > 0 && t.opacity[i] <= 1)) add(int64_t(i), "opacity in (0,1]");
        if (!(t.color_r[i] >= 0 && t.color_r[i] <= 1 && t.color_g[i] >= 0 && t.color_g[i] <= 1 &&
              t.color_b[i] >= 0 && t.color_b[i] <= 1))
            add(int64_t(i), "color in [0,1]");
        const uint32_t p = t.parent[i];
        if (level_of[i] == 0) {
            if (p != kRootParent) add(int64_t(i), "level-0 parent is ROOT");
        } else if (p == kRootParent || p >= n) {
            add(int64_t(i), "parent index in range");
        } else if (level_of[p] + 1 != level_of[i]) {
            add(int64_t(i), "parent level == level - 1");
        }
        const bool is_leaf = t.leaf[i] != 0;
        if (is_leaf == bool(has_child[i])) add(int64_t(i), "leaf iff childless");
    }
    if (n_violations) *n_violations = count;
    return out;
}

std::vector<std::string> validate_camera(const lodgs_camera& c) {
    std::vector<std::string> out;
    if (c.width < 1 || c.height < 1) out.push_back("width, height >= 1");
    if (!(c.fx > 0) || !(c.fy > 0)) out.push_back("fx, fy > 0");
    if (!std::isfinite(c.cx) || !std::isfinite(c.cy)) out.push_back("cx, cy finite");
    if (!(c.znear > 0 && c.znear < c.zfar)) out.push_back("0 < near < far");
    bool finite = true;
    for (double v : c.rotation) finite = finite && std::isfinite(v);
    for (double v : c.translation) finite = finite && std::isfinite(v);
    if (!finite) {
        out.push_back("rotation, translation finite");
        return out;
    }
    const double* r = c.rotation;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double dot = 0;
            for (int k = 0; k < 3; ++k) dot += r[3 * i + k] * r[3 * j + k];
            if (std::abs(dot - (i == j ? 1.0 : 0.0)) > 1e-6) {
                out.push_back("rotation orthonormal");
                i = j = 3;
            }
        }
    return out;
}

std::string join_violations(const std::string& what, const std::vector<std::string>& v,
                            uint64_t total) {
    std::ostringstream ss;
    ss << what << ": ";
    for (size_t i = 0; i < v.size() && i < 8; ++i) {
        if (i) ss << "; ";
        ss << v[i];
    }
    if (total > 8) ss << "; +" << (total - 8) << " more";
    return ss.str();
}

// ---------------------------------------------------------------- camera --
Geom camera_geom(const lodgs_camera& c) {
    Geom g{};
    for (int i = 0; i < 9; ++i) g.rot[i] = c.rotation[i];
    for (int i = 0; i < 3; ++i) g.trans[i] = c.translation[i];
    g.fx = c.fx;
    g.fy = c.fy;
    g.cx = c.cx;
    g.cy = c.cy;
    g.width = c.width;
    g.height = c.height;
    g.znear = c.znear;
    g.zfar = c.zfar;
    auto side = [](double n0, double n1, double n2, double* plane) {
        const double len = std::sqrt(n0 * n0 + n1 * n1 + n2 * n2);
        plane[0] = n0 / len;
        plane[1] = n1 / len;
        plane[2] = n2 / len;
        plane[3] = 0.0;
    };
    for (auto& p : g.planes)
        for (double& v : p) v = 0.0;
    g.planes[0][2] = 1;
    g.planes[0][3] = -g.znear;
    g.planes[1][2] = -1;
    g.planes[1][3] = g.zfar;
    side(g.fx, 0, g.cx, g.planes[2]);
    side(-g.fx, 0, g.width - g.cx, g.planes[3]);
    side(0, g.fy, g.cy, g.planes[4]);
    side(0, -g.fy, g.height - g.cy, g.planes[5]);
    return g;
}

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

void ssim_window(double w[121]) {
    const double sigma = 1.5;
    double sum = 0.0;
    for (int y = 0; y < 11; ++y)
        for (int x = 0; x < 11; ++x) {
            const double dx = x - 11 / 2, dy = y - 11 / 2;
            const double v = std::exp(-(dx * dx + dy * dy) / (2.0 * sigma * sigma));
            w[y * 11 + x] = v;
            sum += v;
        }
    for (int i = 0; i < 121; ++i) w[i] /= sum;
}

}  // namespace fgs
