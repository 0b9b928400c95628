"""B200-native per-frame hot path of arXiv 1809.07986 (tsgm: temporal
Kalman-filtered reduced-space semi-global matching).

The product is the CUDA library ``lib/libtsgm_b200.so`` behind the C-ABI in
``include/tsgm_b200.h``; this package is its Python mirror of the reference's
``tsgm::`` API (see :mod:`.tsgm`)."""
from .tsgm import (  # noqa: F401
    DIAGONAL, NONDIAGONAL, DetectConfig, Engine, EngineConfig, FilterConfig, PipelinedEngine, SgmParams,
    OutlierOptions, StereoCalib, count_outliers, detect_candidate_windows, detect_moving_objects,
    greedy_merge, integral_image, outlier_rate,
    aggregate_paths, build_cost_volume, census_transform, correct, derive_search_ranges,
    disparity_homography, fill_zoom_holes, median_refine, predict, reject_discontinuities,
    relative_motion, sgm_match, step, warp_state_ex, winner_takes_all,
)
