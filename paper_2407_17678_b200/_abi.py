"""ctypes binding of include/s2attn.h (the C ABI of libs2attn.so).

The library must exist in-tree (built by __graft_entry__.build() /
`make -C paper_2407_17678_b200/csrc`); there is no fallback of any kind.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# S2ATTN_VARIANT=<name>: a kernel-tuning build from tools/build_variant.sh
# (paper_2407_17678_b200/variants/<name>/libs2attn.so); unset in production
LIB_PATH = os.path.join(HERE, *(("variants", os.environ["S2ATTN_VARIANT"]) if os.environ.get("S2ATTN_VARIANT") else ()),
                        "libs2attn.so")

S2_OK = 0
S2_ERR_INVALID_ARGUMENT = 1
S2_ERR_CUDA = 2
S2_ERR_UNSUPPORTED = 3
S2_ERR_NO_DEVICE = 4
S2_ERR_OUT_OF_MEMORY = 5
S2_ERR_CONFIG = 6
S2_ERR_BUFFER_TOO_SMALL = 7
S2_MAX_SEGMENTS = 8

S2_DTYPE_BF16 = 0
S2_DTYPE_F32 = 1


class s2_stride_segment(ctypes.Structure):
    _fields_ = [("start_block_distance", ctypes.c_int), ("end_block_distance", ctypes.c_int),
                ("stride", ctypes.c_int), ("num_offsets", ctypes.c_int),
                ("offsets", ctypes.POINTER(ctypes.c_int))]


class s2_pattern_config(ctypes.Structure):
    _fields_ = [("seq_len", ctypes.c_int), ("block_size", ctypes.c_int),
                ("num_heads", ctypes.c_int), ("num_kv_heads", ctypes.c_int),
                ("local_blocks", ctypes.c_int), ("local_stride", ctypes.c_int),
                ("num_segments", ctypes.c_int),
                ("segments", s2_stride_segment * S2_MAX_SEGMENTS)]


class s2_layer_schedule(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int), ("num_dense", ctypes.c_int),
                ("dense_layer_ids", ctypes.POINTER(ctypes.c_int)),
                ("sparse_pattern", s2_pattern_config)]


class s2_config_file(ctypes.Structure):
    _fields_ = [("pattern", s2_pattern_config), ("has_schedule", ctypes.c_int),
                ("schedule", s2_layer_schedule), ("out", ctypes.c_char * 512),
                ("format", ctypes.c_char * 64)]


class s2_flops_report(ctypes.Structure):
    _fields_ = [("dense_flops", ctypes.c_double), ("sparse_flops", ctypes.c_double),
                ("reduction_factor", ctypes.c_double), ("equivalent_context", ctypes.c_double)]


class s2_plan_stats(ctypes.Structure):
    _fields_ = [("num_heads", ctypes.c_int), ("num_kv_heads", ctypes.c_int),
                ("seq_len", ctypes.c_int), ("block_size", ctypes.c_int),
                ("num_blocks", ctypes.c_int), ("nnz_total", ctypes.c_int64),
                ("dense_pairs", ctypes.c_int64), ("max_row_len", ctypes.c_int),
                ("max_col_len", ctypes.c_int), ("fwd_tiles", ctypes.c_int64),
                ("fwd_chunk_visits", ctypes.c_int64), ("bwd_tiles", ctypes.c_int64),
                ("bwd_qtile_visits", ctypes.c_int64)]


class s2_attn_args(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int), ("batch", ctypes.c_int), ("num_heads", ctypes.c_int),
                ("num_kv_heads", ctypes.c_int), ("seq_len", ctypes.c_int),
                ("head_dim", ctypes.c_int), ("scale", ctypes.c_double),
                ("num_splits", ctypes.c_int), ("num_units", ctypes.c_int),
                ("unit_ids", ctypes.POINTER(ctypes.c_int)),
                ("q", ctypes.c_void_p), ("k", ctypes.c_void_p), ("v", ctypes.c_void_p),
                ("out", ctypes.c_void_p), ("lse", ctypes.c_void_p)]


class s2_attn_bwd_args(ctypes.Structure):
    _fields_ = [("fwd", s2_attn_args), ("dout", ctypes.c_void_p), ("dq", ctypes.c_void_p),
                ("dk", ctypes.c_void_p), ("dv", ctypes.c_void_p)]


# Every symbol include/s2attn.h declares: name -> (restype, argtypes).
_P = ctypes.c_void_p
_I = ctypes.c_int
_I64P = ctypes.POINTER(ctypes.c_int64)
_IP = ctypes.POINTER(ctypes.c_int)
_CFG = ctypes.POINTER(s2_pattern_config)
_SCH = ctypes.POINTER(s2_layer_schedule)
_SZP = ctypes.POINTER(ctypes.c_size_t)
_DP = ctypes.POINTER(ctypes.c_double)
SIGNATURES = {
    "s2_last_error": (ctypes.c_char_p, []),
    "s2_abi_version": (_I, []),
    "s2_set_sm_reserve": (_I, [_I]),
    "s2_make_single_stride_config": (_I, [_I, _I, _I, _I, _I, _I, _CFG]),
    "s2_pattern_validate": (_I, [_CFG]),
    "s2_pattern_num_blocks": (_I, [_CFG]),
    "s2_pattern_offset_for": (_I, [_CFG, _I, _I, _IP]),
    "s2_layout_nnz": (_I, [_CFG, _I, _I64P]),
    "s2_layout_build_csr": (_I, [_CFG, _I, _IP, _IP]),
    "s2_layout_build_csc": (_I, [_CFG, _I, _IP, _IP]),
    "s2_layout_evict_after": (_I, [_CFG, _I, _IP]),
    "s2_layout_kv_efficient": (_I, [_CFG, _I, _IP]),
    "s2_csr_validate": (_I, [_I, _IP, _IP, ctypes.c_int64]),
    "s2_plan_create": (_I, [_CFG, ctypes.POINTER(_P)]),
    "s2_plan_create_from_csr": (_I, [_I, _I, _I, _I, ctypes.POINTER(_IP), ctypes.POINTER(_IP),
                                     ctypes.POINTER(_P)]),
    "s2_plan_destroy": (None, [_P]),
    "s2_plan_get_stats": (_I, [_P, ctypes.POINTER(s2_plan_stats)]),
    "s2_plan_head_nnz": (_I, [_P, _I, _I64P]),
    "s2_plan_fwd_tiles": (_I, [_P, _IP, _I64P, _I64P, ctypes.POINTER(ctypes.c_int32),
                               ctypes.POINTER(ctypes.c_uint32)]),
    "s2_plan_bwd_tiles": (_I, [_P, _I64P, _I64P, _I64P, _I64P]),
    "s2_attn_fwd": (_I, [_P, ctypes.POINTER(s2_attn_args), _P]),
    "s2_attn_fwd_peers": (_I, [_P, ctypes.POINTER(s2_attn_args), _I, ctypes.POINTER(ctypes.c_void_p),
                               ctypes.POINTER(ctypes.c_void_p), _P, _I, _P]),
    "s2_attn_bwd_workspace_size": (_I, [_P, ctypes.POINTER(s2_attn_bwd_args),
                                        ctypes.POINTER(ctypes.c_size_t)]),
    "s2_attn_bwd": (_I, [_P, ctypes.POINTER(s2_attn_bwd_args), _P, ctypes.c_size_t, _P]),
    "s2_attn_fwd_bwd_host_workspace_size": (_I, [_P, ctypes.POINTER(s2_attn_bwd_args), _I,
                                                 ctypes.POINTER(ctypes.c_size_t)]),
    "s2_attn_fwd_bwd_host": (_I, [_P, ctypes.POINTER(s2_attn_bwd_args), _I, _P, ctypes.c_size_t, _P]),
    "s2_kvcache_create": (_I, [_P, _I, _I, _I, ctypes.POINTER(_P)]),
    "s2_kvcache_destroy": (None, [_P]),
    "s2_kvcache_length": (_I, [_P, _IP]),
    "s2_kvcache_bytes": (_I, [_P, _I64P, _I64P]),
    "s2_kvcache_retained_tokens": (_I, [_P, _I, _I64P]),
    "s2_kvcache_prefill": (_I, [_P, _P, _P, _I, _P]),
    "s2_kvcache_append": (_I, [_P, _P, _P, _P]),
    "s2_attn_decode_workspace_size": (_I, [_P, ctypes.POINTER(ctypes.c_size_t)]),
    "s2_attn_decode": (_I, [_P, _P, _P, _P, ctypes.c_double, _P, ctypes.c_size_t, _P]),
    "s2_attn_decode_bytes": (_I, [_P, _I64P]),
    "s2_plan_unit_weights": (_I, [_P, _I, _I64P]),
    "s2_partition_lpt": (_I, [_I, _I64P, _I, _IP, _I64P]),
    "s2_plan_fwd_flops": (_I, [_P, _I, _I, ctypes.POINTER(ctypes.c_double),
                               ctypes.POINTER(ctypes.c_double)]),
    "s2_random_tensors": (_I, [_I, _I, _I, ctypes.c_uint64, ctypes.POINTER(ctypes.c_float),
                              ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]),
    "s2_device_count": (_I, [_IP]),
    "s2_device_malloc": (_I, [ctypes.POINTER(_P), ctypes.c_size_t]),
    "s2_device_free": (_I, [_P]),
    "s2_memcpy_h2d": (_I, [_P, _P, ctypes.c_size_t, _P]),
    "s2_memcpy_d2h": (_I, [_P, _P, ctypes.c_size_t, _P]),
    "s2_stream_synchronize": (_I, [_P]),
    "s2_pattern_to_json": (_I, [_CFG, ctypes.c_char_p, ctypes.c_size_t, _SZP]),
    "s2_pattern_from_json": (_I, [ctypes.c_char_p, _CFG, _IP, _I]),
    "s2_pattern_hash": (_I, [_CFG, ctypes.POINTER(ctypes.c_uint64)]),
    "s2_csr_to_json": (_I, [_I, _I, _IP, _IP, ctypes.c_char_p, ctypes.c_size_t, _SZP]),
    "s2_csr_from_json": (_I, [ctypes.c_char_p, _IP, _IP, _IP, _I, _IP, ctypes.c_int64, _I64P]),
    "s2_schedule_validate": (_I, [_SCH]),
    "s2_schedule_to_json": (_I, [_SCH, ctypes.c_char_p, ctypes.c_size_t, _SZP]),
    "s2_schedule_from_json": (_I, [ctypes.c_char_p, _CFG, _SCH, _IP, _I, _IP, _I]),
    "s2_config_file_load": (_I, [ctypes.c_char_p, ctypes.POINTER(s2_config_file), _IP, _I, _IP, _I]),
    "s2_equivalent_context_length": (_I, [ctypes.c_double] * 3 + [_DP]),
    "s2_analytic_flops_reduction": (_I, [ctypes.c_double] * 3 + [_DP]),
    "s2_speedup_upper_bound": (_I, [_I, ctypes.c_double, ctypes.c_double, _DP]),
    "s2_exact_flops": (_I, [_CFG, _I, ctypes.POINTER(s2_flops_report), _I64P]),
    "s2_simulate_decode_cache": (_I, [_CFG, _I, _I, _IP, _I64P, _IP, _I64P, _DP]),
    "s2_kv_reduction": (_I, [_SCH, _DP]),
    "s2_layers_create": (_I, [_SCH, ctypes.POINTER(_P)]),
    "s2_layers_destroy": (None, [_P]),
    "s2_layers_plan": (_I, [_P, _I, ctypes.POINTER(_P), _IP]),
    "s2_layers_fwd": (_I, [_P, _I, ctypes.POINTER(s2_attn_args), _P]),
    "s2_layers_bwd": (_I, [_P, _I, ctypes.POINTER(s2_attn_bwd_args), _P, ctypes.c_size_t, _P]),
    "s2_profile_enable": (_I, [_I]),
    "s2_profile_collect": (_I, [_I, ctypes.c_char_p, ctypes.POINTER(ctypes.c_double), _IP, _IP]),
}


class S2Error(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[s2 status {code}] {msg}")
        self.code = code


class S2InvalidArgument(S2Error, ValueError):
    """Maps the reference's std::invalid_argument."""


class S2Unsupported(S2Error, NotImplementedError):
    pass


class S2ConfigError(S2Error):
    """Maps load_config_file's std::runtime_error (serialize.cpp:123-146)."""


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() or "
                f"`make -C paper_2407_17678_b200/csrc` (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("S2ATTN_VARIANT") and not hasattr(L, name):
                continue  # a tuning build of an older tree may predate a symbol
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc):
    if rc == S2_OK:
        return
    msg = lib().s2_last_error().decode()
    if rc == S2_ERR_INVALID_ARGUMENT:
        raise S2InvalidArgument(rc, msg)
    if rc == S2_ERR_UNSUPPORTED:
        raise S2Unsupported(rc, msg)
    if rc == S2_ERR_CONFIG:
        raise S2ConfigError(rc, msg)
    raise S2Error(rc, msg)
