"""B200-native sparse-convolution engine (Minuet Map + GMaS) behind the reference SC-layer API.

The compute path is libsconv_b200.so (hand-written sm_100a CUDA behind a C ABI,
include/sconv_b200.h); this package is its Python binding. No CPU fallback exists.
"""
from .sconv import (  # noqa: F401
    BF16, DATAFLOW_AUTO, DATAFLOW_FUSED, DATAFLOW_GMAS, F16, F32, GROUP_MAP_ORDER, GROUP_SORTED, MAP_HASH, MAP_SORTED, MAP_SORTED_SPEC, MEM_DEVICE, MEM_HOST, Context, CudaError, ExecCfg,
    InvalidArgument, KernelMap, LogicError, MapCfg, OutOfRange, PointCloud, SconvError, Weights,
    build_kernel_map_sorted, build_kernel_map_sorted_explicit, cloud_file_info, exec_cfg, FILE_MPC, FILE_XYZ, generate_synthetic, generate_weights, layer_forward, layer_forward_device,
    load, load_cloud, map_cfg, read_cloud, write_mpc, write_xyz, plan_groups, sc_layer_forward, theoretical_hyperparams, tune_layer, voxelize, weight_offsets,
)

__all__ = [n for n in dir() if not n.startswith("_")]
