// ref_ldgs_tool -- TEST INFRASTRUCTURE ONLY.  A tiny native driver over the
// reference library compiled in place (oracle/_ref/libref_lodgs.so) for the
// LDGS v1 scene-file tests: the reference's save_scene / load_scene
// (scene_io.cpp:200-226) run in a native process (iostreams of the
// statically linked libstdc++ misbehave when the library is dlopen'ed from
// Python).
//
//   ref_ldgs_tool save <path> nx ny scene_seed depth build_seed
//       build_tree(generate_synthetic_scene(spec)) -> save_scene(path)
//   ref_ldgs_tool load <path>
//       load_scene(path): prints "OK <nodes> <levels> <fnv64 of the SoA arrays>"
//       or "ERR <IoError|FormatError|ValidationError> <message>"
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "lodgs/scene_io.hpp"
#include "lodgs/tree_builder.hpp"

using namespace lodgs;

namespace {
uint64_t fnv(uint64_t h, const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}
}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) return 64;
    const std::string cmd = argv[1], path = argv[2];
    if (cmd == "save" && argc == 8) {
        SyntheticSceneSpec s;
        s.nx = uint32_t(std::atoi(argv[3]));
        s.ny = uint32_t(std::atoi(argv[4]));
        s.seed = std::strtoull(argv[5], nullptr, 10);
        TreeBuildConfig c;
        c.depth = uint32_t(std::atoi(argv[6]));
        c.seed = std::strtoull(argv[7], nullptr, 10);
        save_scene(build_tree(generate_synthetic_scene(s), c), path);
        std::printf("SAVED\n");
        return 0;
    }
    if (cmd == "load") {
        try {
            const LoDTree t = load_scene(path);
            uint64_t h = 1469598103934665603ull;
            for (const auto* v : {&t.mean_x, &t.mean_y, &t.mean_z, &t.scale_x, &t.scale_y,
                                  &t.scale_z, &t.quat_w, &t.quat_x, &t.quat_y, &t.quat_z,
                                  &t.opacity, &t.color_r, &t.color_g, &t.color_b})
                h = fnv(h, v->data(), v->size() * 4);
            h = fnv(h, t.parent.data(), t.parent.size() * 4);
            h = fnv(h, t.leaf.data(), t.leaf.size());
            std::printf("OK %zu %zu %llu\n", t.node_count(), t.level_count(),
                        (unsigned long long)h);
        } catch (const IoError& e) {
            std::printf("ERR IoError %s\n", e.what());
        } catch (const FormatError& e) {
            std::printf("ERR FormatError %s\n", e.what());
        } catch (const ValidationError& e) {
            std::printf("ERR ValidationError %s\n", e.what());
        }
        return 0;
    }
    return 64;
}
