// host_util.h -- host-side utilities shared by the C ABI and the C++ API.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lodgs_gpu.h"
#include "common.cuh"

namespace fgs {

// Carries a lodgs_status code across the C ABI.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

std::vector<std::string> validate_tree(const lodgs_tree_view& t, uint64_t* n_violations);
// The tree-level rules of validate_tree (scene.cpp:93-116), with the same
// messages; returns false when the per-node rules must not run (bad arrays,
// bad level offsets, empty tree).  Per-node rules then run on the device.
bool validate_tree_header(const lodgs_tree_view& t, std::vector<std::string>& out,
                          uint64_t& count);
// Message of per-node rule bit k (ingest.cu k_validate_nodes order).
const char* node_rule_name(int k);
std::vector<std::string> validate_camera(const lodgs_camera& c);
std::string join_violations(const std::string& what, const std::vector<std::string>& v,
                            uint64_t total);
Geom camera_geom(const lodgs_camera& c);
// metrics.cpp:136-154 SsimWindow: normalised 11x11 Gaussian, sigma 1.5
void ssim_window(double w[121]);

}  // namespace fgs
