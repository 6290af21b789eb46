/* lodgs_synth.h -- benchmark INPUT generation (not the hot path, not in the
 * renderer library): the reference's synthetic scene generator + LoD builder
 * (tree_builder.hpp:11-33, tree_builder.cpp:75-174) and CameraPath::sample
 * (camera_path.cpp:126-180), restated bit for bit.  Library:
 * paper_2603_23891_b200/_lib/liblodgs_synth.so.  Status codes as lodgs_gpu.h;
 * lodgs_synth_last_error() holds the message. */
#ifndef LODGS_SYNTH_H
#define LODGS_SYNTH_H

#include "lodgs_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

LODGS_API const char *lodgs_synth_last_error(void);

/* camera_path.cpp:126-180: frames = sum(samples)+1; out holds that many. */
LODGS_API int lodgs_camera_path_sample(const lodgs_camera *keyframes, uint32_t n_keyframes,
                             const uint32_t *samples, lodgs_camera *out, uint64_t out_cap,
                             uint64_t *n_frames);

/* tree_builder.hpp:11-27 configs. */
typedef struct lodgs_synthetic_spec {
    uint32_t nx, ny;
    float spacing;
    float scale_min, scale_max;
    float opacity_min, opacity_max;
    uint64_t seed;
    uint32_t congestion;
} lodgs_synthetic_spec;

typedef struct lodgs_build_config {
    uint32_t depth;
    float shrink_factor;
    uint32_t children_per_node;
    uint64_t seed;
} lodgs_build_config;

/* Writable SoA arrays for tree construction (capacity = n_nodes). */
typedef struct lodgs_tree_buffers {
    float *mean_x, *mean_y, *mean_z;
    float *scale_x, *scale_y, *scale_z;
    float *quat_w, *quat_x, *quat_y, *quat_z;
    float *opacity;
    float *color_r, *color_g, *color_b;
    uint32_t *parent;
    uint8_t *leaf;
    uint32_t *level_offsets; /* capacity depth+1 */
} lodgs_tree_buffers;

/* generate_synthetic_scene + build_tree (tree_builder.cpp:75-174): first call
 * with out == NULL to learn n_nodes / n_levels, then with buffers. */
LODGS_API int lodgs_build_synthetic_tree(const lodgs_synthetic_spec *spec, const lodgs_build_config *cfg,
                               lodgs_tree_buffers *out, uint64_t *n_nodes, uint32_t *n_levels);

#ifdef __cplusplus
}
#endif

#endif /* LODGS_SYNTH_H */
