"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This package holds NO arithmetic of the method (no clipping, no area, no IoU):
only random box/polygon parameters and their vertex coordinates, rounded once
to float32.  See DESIGN.md "Input recipe" and SURVEY.md §8(d).
"""
from .generators import (  # noqa: F401
    CONFIGS,
    Polys,
    PairBatch,
    Scene,
    BoxPairBatch,
    boxes_to_polys,
    gen_box_pairs,
    gen_cfg1_pairs,
    gen_cfg2_scene,
    gen_cfg3_pairs,
    gen_cfg4_pairs,
    gen_cfg5_scene,
    gen_config,
    gen_quad_pairs,
    gen_thin_pairs,
    seed_for,
)
