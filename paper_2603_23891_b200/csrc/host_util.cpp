// host_util.cpp -- host-side scene utilities of the lodgs API, restated in
// C++ for the B200 build: tree / camera validation (scene.cpp:89-199) and
// CameraGeom::make (projection.cpp:11-38).  None of this is per-frame GPU work;
// it runs once per upload / per camera.  (Input generation -- the synthetic
// scene generator and camera paths -- lives in synth.cpp, a separate library.)
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
