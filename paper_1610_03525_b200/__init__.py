"""B200-native fBm heightmap path (arXiv 1610.03525 polynomial terrain noise).

Drop-in for the reference generator API (terrain/fbm.hpp:538-685) and the
fractal-analysis pass (terrain/analysis.hpp) over the C-ABI in
include/polyterrain_b200.h, implemented by hand-written sm_100a kernels in
paper_1610_03525_b200/csrc/.  No CPU fallback.
"""
from .fbm import (  # noqa: F401
    BoxCountReport, DeviceError, FbmConfig, Heightmap, IoError, LinearFit, Method, NumericalError,
    OctaveSpec, ValidationError, box_count_device, box_count_mask_device, coastline_mask_device,
    default_box_sizes, ffma_peak_tflops, generate3d_device, generate_batch_device, generate_heightmap,
    generate_into, generate_into_device, generate_rect_device, generate_region, linear_fit,
    method_name, normalize_map, octave_spec, parse_method, upper_median_device, variogram_device,
    variogram_dimension, TextureKind, texture_device, norm_map_device, encode_pgm16, encode_png16, write_pgm16, write_png16,
)
