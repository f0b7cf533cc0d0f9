"""B200-native SS-CGA delay-Doppler equalizer (drop-in for ddlink's hot path).

Reference: arxiv/paper_2604_02266, package `ddlink` (/root/reference/pkg).
The drop-in names below keep the reference's signatures, layouts and errors;
their arithmetic runs in hand-written sm_100a CUDA kernels (libddb.so, C ABI
in include/ddb.h).  `SsCgaSolver` is the batched device API.
"""

from .batch import HostPipeline, PathBatch, SolveResult, SsCgaSolver, bits_per_symbol, pack_labels
from .equalize import CgaConfig, CgaTrace, cga_equalize, get_precision, set_precision
from .pilot import build_twist_kernel, default_pilot_amplitude, estimate_heff, make_pilot_frame
from .grid import (
    Constellation,
    GridConfig,
    ber,
    check_frame,
    check_signal,
    flatten,
    hard_demod,
    make_constellation,
    make_constellation_ext,
    modulate,
    unflatten,
)
from .sparse import (
    DominantPath,
    EmptyChannel,
    StructuredSparseChannel,
    build_ss_channel,
    coefficient,
    detect_paths,
    forward_index,
    inverse_index,
    ss_mvm,
    ss_mvm_hermitian,
)
from .zak import build_zak_kernel, dzt_device, dzt_gemm
from .dense import build_dense_hdd, lmmse_equalize, receive_lmmse, threshold_frame
from .channel import (
    ChannelBatch,
    PathSet,
    PathSpec,
    add_awgn,
    add_awgn_device,
    apply_channel,
    apply_channel_device,
    draw_veha,
    draw_veha_batch,
    idzt,
    idzt_device,
    make_path,
    modulate_device,
)

__all__ = [
    "HostPipeline", "PathBatch", "SolveResult", "SsCgaSolver", "bits_per_symbol", "pack_labels",
    "CgaConfig", "CgaTrace", "cga_equalize", "get_precision", "set_precision",
    "Constellation", "GridConfig", "ber", "check_frame", "check_signal", "flatten", "hard_demod",
    "make_constellation", "make_constellation_ext", "modulate", "unflatten",
    "DominantPath", "EmptyChannel", "StructuredSparseChannel", "build_ss_channel", "coefficient",
    "detect_paths", "forward_index", "inverse_index", "ss_mvm", "ss_mvm_hermitian",
    "build_twist_kernel", "default_pilot_amplitude", "estimate_heff", "make_pilot_frame",
    "build_zak_kernel", "dzt_device", "dzt_gemm",
    "ChannelBatch", "PathSet", "PathSpec", "add_awgn", "add_awgn_device", "apply_channel", "apply_channel_device",
    "draw_veha", "draw_veha_batch", "idzt", "idzt_device", "make_path", "modulate_device",
    "build_dense_hdd", "lmmse_equalize", "receive_lmmse", "threshold_frame",
]

__version__ = "0.1.0"
