"""The C-ABI library loads without a GPU and exports every symbol include/*.h declares."""
import ctypes
import os
import re

import paper_2407_17678_b200 as s2
from paper_2407_17678_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "s2attn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(s2_[a-z0-9_]+)\s*\(", src))
    return sorted(n for n in names if n != "s2_stream_t")


def test_every_declared_symbol_is_exported_and_bound():
    lib = ctypes.CDLL(_abi.LIB_PATH)
    decl = declared_functions()
    assert len(decl) > 30
    for name in decl:
        assert hasattr(lib, name), f"{name} declared in s2attn.h but not exported"
        assert name in _abi.SIGNATURES, f"{name} has no ctypes binding"


def test_abi_version_and_error_string():
    L = s2.lib()
    assert L.s2_abi_version() == 1
    assert L.s2_pattern_validate(None) == _abi.S2_ERR_INVALID_ARGUMENT
    assert b"null" in L.s2_last_error()


def test_host_layout_calls_work_without_gpu():
    cfg = s2.make_s2_config(4096, 8, vert_stride=4)
    plan = s2.Plan.from_config(cfg)
    st = plan.stats()
    assert st["nnz_total"] == sum(s2.build_csr(cfg, h).nnz() for h in range(8))
    a, d = plan.fwd_flops(2, 128)
    assert a < d


def test_device_calls_fail_loudly_without_gpu():
    """No CPU fallback: without a device the forward reports an error."""
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    t = s2.AttentionTensors.random(2, 16, 8, 1)
    with pytest.raises(s2.S2Error):
        s2.streaming_sharded_attention(t, s2.build_all_csr(s2.make_single_stride_config(16, 8, 2, 1, 1)), 8)


def test_fwd_peers_argument_errors_without_a_device():
    """s2_attn_fwd_peers validates its exchange arguments before any device work."""
    import ctypes

    import paper_2407_17678_b200 as s2
    from paper_2407_17678_b200 import _abi

    plan = s2.Plan.from_config(s2.make_s2_config(256, 2, block_size=64, local_blocks=1, vert_stride=2))
    L = _abi.lib()
    a = _abi.s2_attn_args()
    bufs = (ctypes.c_void_p * 1)(None)
    for n in (0, 9):
        assert L.s2_attn_fwd_peers(plan.handle, ctypes.byref(a), n, bufs, bufs, None, 1, None) == 1
        assert b"num_peers" in L.s2_last_error()
    assert L.s2_attn_fwd_peers(plan.handle, ctypes.byref(a), 1, bufs, bufs, None, 1, None) == 1
    assert b"required" in L.s2_last_error()
