"""ctypes binding of libvcnn_cuda.so (the C ABI in include/vcnn_cuda.h).

The library is built in-tree by `make lib` (or __graft_entry__.build()).  There
is no fallback: if the shared object is missing, importing anything that needs
it raises immediately.
"""
import ctypes as C
import os

from .errors import STATUS_TO_ERROR, VcnnError

_HERE = os.path.dirname(os.path.abspath(__file__))
# VCNN_LIB_PATH: an alternative in-tree build (e.g. the phase-timing build of
# scripts/phase_timing.py); default the product library
LIB_PATH = os.environ.get("VCNN_LIB_PATH") or os.path.join(_HERE, "libvcnn_cuda.so")

c_int = C.c_int
c_i64 = C.c_int64
c_float = C.c_float
c_double = C.c_double
c_vp = C.c_void_p
P_i64 = C.POINTER(C.c_int64)
P_int = C.POINTER(C.c_int)
P_float = C.POINTER(C.c_float)


class ConvGeometryC(C.Structure):
    """vcnn_conv_geometry == ConvGeometry (vectorize.hpp:13-42)."""

    _fields_ = [(n, c_int) for n in
                ("in_h", "in_w", "channels", "batch", "kh", "kw", "stride", "out_h", "out_w")]


class PoolGeometryC(C.Structure):
    """vcnn_pool_geometry == PoolGeometry (vectorize.hpp:134-162)."""

    _fields_ = [(n, c_int) for n in
                ("in_h", "in_w", "channels", "batch", "ph", "pw", "stride", "mode", "out_h",
                 "out_w")]


class LayerSpecC(C.Structure):
    """vcnn_layer_spec == one LayerSpec (network.hpp:12-32)."""

    _fields_ = [(n, c_int) for n in
                ("kind", "units", "kh", "kw", "stride", "pool_mode", "pool_bias", "act")]


class NetSpecC(C.Structure):
    """vcnn_net_spec == NetworkSpec (network.hpp:37-73)."""

    _fields_ = [("in_h", c_int), ("in_w", c_int), ("in_c", c_int), ("nlayers", c_int),
                ("layers", C.POINTER(LayerSpecC)), ("loss", c_int), ("seed", C.c_uint64)]


# name -> argtypes (restype is int unless listed in _RESTYPES)
_SIGS = {
    "vcnn_abi_version": [],
    "vcnn_last_error": [],
    "vcnn_device_info": [P_int, P_int, P_int],
    "vcnn_launch_count": [],
    "vcnn_conv_geometry_init": [C.POINTER(ConvGeometryC)] + [c_int] * 7,
    "vcnn_pool_geometry_init": [C.POINTER(PoolGeometryC)] + [c_int] * 8,
    "vcnn_net_spec_chain": [C.POINTER(NetSpecC), P_int],
    "vcnn_synth_bench_data": [C.POINTER(NetSpecC), c_int, C.c_uint64, c_vp, c_vp, c_vp],
    "vcnn_matmul": [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_int, c_vp],
    "vcnn_matmul_transB": [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_int, c_vp],
    "vcnn_gemm": [c_int, c_int, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp,
                  c_int, c_int, c_vp],
    "vcnn_accumulate_by_index": [c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_int, c_vp, c_vp],
    "vcnn_accumulate_max_arg": [c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp],
    "vcnn_im2col": [C.POINTER(ConvGeometryC), c_vp, c_vp, c_vp],
    "vcnn_col2im": [C.POINTER(ConvGeometryC), c_vp, c_vp, c_vp],
    "vcnn_col2im_map": [C.POINTER(ConvGeometryC), c_vp, c_vp, c_vp],
    "vcnn_pool_map": [C.POINTER(PoolGeometryC), c_vp, c_vp, c_vp],
    "vcnn_pool_forward": [C.POINTER(PoolGeometryC), c_vp, c_vp, c_vp, c_vp],
    "vcnn_pool_backward": [C.POINTER(PoolGeometryC), c_int, c_vp, c_vp, c_vp, c_vp],
    "vcnn_activation_forward": [c_i64, c_int, c_vp, c_vp, c_vp],
    "vcnn_activation_backward": [c_i64, c_int, c_vp, c_vp, c_vp],
    "vcnn_conv_forward": [C.POINTER(ConvGeometryC), c_int, c_vp, c_vp, c_vp, c_int, c_int, c_vp,
                          c_vp],
    "vcnn_conv_backward": [C.POINTER(ConvGeometryC), c_int, c_vp, c_vp, c_vp, c_vp, c_int, c_int,
                           c_vp, c_vp, c_vp, c_vp],
    "vcnn_full_forward": [c_int, c_int, c_int, c_vp, c_vp, c_vp, c_int, c_int, c_vp, c_vp],
    "vcnn_full_backward": [c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_vp, c_vp,
                           c_vp, c_vp],
    "vcnn_pool_layer_forward": [C.POINTER(PoolGeometryC), c_vp, c_vp, c_int, c_vp, c_vp, c_vp],
    "vcnn_pool_layer_backward": [C.POINTER(PoolGeometryC), c_int, c_vp, c_int, c_vp, c_vp, c_vp,
                                 c_vp, c_vp],
    "vcnn_loss_forward": [c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp],
    "vcnn_loss_backward": [c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp],
    "vcnn_loss_fused": [c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "vcnn_sgd_step": [c_i64, c_vp, c_vp, c_vp, c_float, c_float, c_float, c_vp],
    "vcnn_net_create": [C.POINTER(NetSpecC), c_int, c_int, C.POINTER(c_vp)],
    "vcnn_net_destroy": [c_vp],
    "vcnn_net_num_params": [c_vp],
    "vcnn_net_param_layout": [c_vp, P_i64, P_i64, P_i64, P_i64],
    "vcnn_net_layer_out_size": [c_vp, c_int, P_i64],
    "vcnn_net_set_stream": [c_vp, c_vp],
    "vcnn_net_set_pool_backward_mode": [c_vp, c_int],
    "vcnn_net_set_precision": [c_vp, c_int],
    "vcnn_net_set_fusion": [c_vp, c_int],
    "vcnn_copy_h2d": [c_vp, c_vp, C.c_size_t],
    "vcnn_net_train_epoch": [c_vp, c_vp, c_vp, c_vp, c_int, c_vp, c_int, c_float, c_float, c_vp],
    "vcnn_net_set_trace": [c_vp, c_int],
    "vcnn_net_get_params": [c_vp, c_vp],
    "vcnn_net_set_params": [c_vp, c_vp],
    "vcnn_net_get_grads": [c_vp, c_vp],
    "vcnn_net_get_velocity": [c_vp, c_vp],
    "vcnn_net_set_velocity": [c_vp, c_vp],
    "vcnn_net_device_buffers": [c_vp, C.POINTER(c_vp), C.POINTER(c_vp), C.POINTER(c_vp)],
    "vcnn_net_params_updated": [c_vp],
    "vcnn_net_set_nonfinite_guard": [c_vp, c_int],
    "vcnn_dp_unique_id": [c_vp],
    "vcnn_dp_init": [c_vp, c_int, c_int, c_vp, C.POINTER(c_vp)],
    "vcnn_dp_create": [c_vp, c_int, c_int, C.POINTER(c_vp)],
    "vcnn_dp_handle": [c_vp, c_vp],
    "vcnn_dp_connect": [c_vp, c_vp, c_vp],
    "vcnn_dp_group": [c_vp, c_int, c_int, c_vp],
    "vcnn_dp_group_train_step": [c_vp, c_int, c_vp, c_float, c_float],
    "vcnn_dp_set_mode": [c_vp, c_int],
    "vcnn_dp_get_mode": [c_vp, P_int],
    "vcnn_dp_set_shards": [c_vp, c_vp],
    "vcnn_dp_allreduce_sgd": [c_vp, c_float, c_float],
    "vcnn_dp_train_step": [c_vp, c_int, c_float, c_float],
    "vcnn_dp_status": [c_vp],
    "vcnn_dp_destroy": [c_vp],
    "vcnn_net_input_buffers": [c_vp, C.POINTER(c_vp), C.POINTER(c_vp), C.POINTER(c_vp)],
    "vcnn_net_set_batch_device": [c_vp, c_int, c_vp, c_vp, c_vp],
    "vcnn_net_set_batch_ring": [c_vp, c_int, c_int, c_vp, c_i64, c_vp, c_i64],
    "vcnn_net_train_steps": [c_vp, c_int, c_int, C.c_float, C.c_float],
    "vcnn_net_forward_backward": [c_vp, c_int],
    "vcnn_net_forward": [c_vp, c_int],
    "vcnn_net_sgd_step": [c_vp, c_float, c_float, c_float],
    "vcnn_net_train_step": [c_vp, c_int, c_float, c_float],
    "vcnn_net_train_step_host": [c_vp, c_int, c_vp, c_vp, c_vp, c_float, c_float, P_float],
    "vcnn_net_train_host_stream": [c_vp, c_int, c_int, c_vp, C.c_int64, c_vp, c_vp, C.c_int64,
                                   c_float, c_float, c_vp],
    "vcnn_net_forward_host": [c_vp, c_int, c_vp, c_vp],
    "vcnn_net_enable_graph": [c_vp, c_int],
    "vcnn_net_get_loss": [c_vp, P_float],
    "vcnn_net_get_output": [c_vp, c_vp],
    "vcnn_net_get_layer_output": [c_vp, c_int, c_vp],
    "vcnn_net_get_pool_arg": [c_vp, c_int, c_vp],
    "vcnn_net_get_layer_grad": [c_vp, c_int, c_vp],
    "vcnn_net_kernels_per_step": [c_vp, P_int],
    "vcnn_net_enable_breakdown": [c_vp, c_int],
    "vcnn_net_read_breakdown": [c_vp, C.POINTER(c_double)],
    "vcnn_net_read_op_timing": [c_vp, C.POINTER(c_double), P_i64],
}
_RESTYPES = {"vcnn_last_error": C.c_char_p, "vcnn_launch_count": c_i64,
             "vcnn_net_num_params": c_i64}

_lib = None


def lib():
    """Load libvcnn_cuda.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: build it with `make lib` (or "
                "__graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, argtypes in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, c_int)
        _lib = L
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def check(status):
    """Raise the reference exception type for a non-zero vcnn_status."""
    if status:
        msg = lib().vcnn_last_error()
        msg = msg.decode() if msg else ""
        raise STATUS_TO_ERROR.get(status, VcnnError)(msg or f"vcnn status {status}")
    return status
