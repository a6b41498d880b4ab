"""Seeded input generators (slides, weights, workload records).

Shared by the oracle side and the CUDA side; holds none of the method's
arithmetic (see DESIGN.md §4 for the recipe)."""
from .arch import (CLASSES, SCALE_CODES_4, TASKS_6, THETA_LEN, HEAD_WIDTH, arch_dict,  # noqa: F401
                   arch_string, blob_layout, channels, make_weights, param_count, split_blob,
                   workload, Workload)
from .synth import geometry, make_slide, render, sha256, blank_slide, random_tiles  # noqa: F401
