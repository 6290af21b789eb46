"""Per-stage device times of cfg-4 frames (50M-node tree, 3840x2160, fx 2000) at a few
altitudes, three-sigma: where a 4K frame spends its time."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import topdown_camera  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402

tree = L.build_synthetic_tree(nx=103, ny=104, seed=1, depth=4, build_seed=7)
with L.GpuScene(tree) as s:
    alts = [float(a) for a in os.environ.get("CFG4_ALTS", "400,300,200,110").split(",")]
    for alt in alts:
        cam = topdown_camera(3840, 2160, 2000.0, alt)
        for _ in range(3):
            out = s.render(cam, L.FilterConfig(3.0), L.ShrinkMode.three_sigma(),
                           L.RenderOptions(stage_timing=True))
        st = out.stats
        print(f"alt {alt}: sel {st.n_selected} pairs {st.n_pairs} big {st.big_tiles} "
              f"filter {st.t_calc_ms + st.t_sync_ms:.3f} (calc {st.t_calc_ms:.3f} sync "
              f"{st.t_sync_ms:.3f}) prep {st.t_prepr_ms:.3f} sort {st.t_sort_ms:.3f} "
              f"blend {st.t_alpha_ms:.3f} ms", flush=True)

    # tile-size distribution of the lowest frame: what the big-bucket sort sees
    import numpy as np
    nt = ((3840 + 15) // 16) * ((2160 + 15) // 16)
    _, pt = s.read_counts(int(st.n_selected), nt)
    pt = pt.astype(np.int64)
    for cap in (2048, 4096, 16384):
        big = pt[pt > cap]
        print(f"tiles > {cap}: {big.size}, keys {big.sum()} ({big.sum() / max(1, pt.sum()):.1%})")
    print("percentiles 50/90/99/max:", np.percentile(pt, [50, 90, 99]).tolist(), pt.max())
