"""tcgen05 building-block probes (SS and TS MMA, SW128 TMA tiles) vs torch."""
import ctypes
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "cuda", "libumma_probe.so")


def _lib():
    src = os.path.join(HERE, "cuda", "umma_probe.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(
            ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
             "-Xcompiler", "-fPIC", "-shared", "-o", SO, src])
    lib = ctypes.CDLL(SO)
    lib.probe_last_error.restype = ctypes.c_char_p
    return lib


@pytest.mark.gpu
@pytest.mark.parametrize("N,K", [(128, 128), (64, 128), (128, 64), (256, 64)])
def test_probe_ss(N, K):
    import torch

    lib = _lib()
    torch.manual_seed(0)
    A = torch.randn(128, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    D = torch.zeros(128, N, device="cuda")
    rc = lib.probe_ss(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()), N, K,
                      ctypes.c_void_p(D.data_ptr()))
    assert rc == 0, lib.probe_last_error()
    ref = A.float() @ B.float().T
    torch.testing.assert_close(D, ref, rtol=1e-3, atol=1e-3)


@pytest.mark.gpu
@pytest.mark.parametrize("KK,Dv", [(128, 128), (64, 128), (128, 64)])
def test_probe_ts(KK, Dv):
    import torch

    lib = _lib()
    torch.manual_seed(1)
    P = torch.rand(128, KK, device="cuda")
    V = torch.randn(KK, Dv, device="cuda").to(torch.bfloat16)
    O = torch.zeros(128, Dv, device="cuda")
    rc = lib.probe_ts(ctypes.c_void_p(P.data_ptr()), ctypes.c_void_p(V.data_ptr()), KK, Dv,
                      ctypes.c_void_p(O.data_ptr()))
    assert rc == 0, lib.probe_last_error()
    ref = P.to(torch.bfloat16).float() @ V.float()
    torch.testing.assert_close(O, ref, rtol=1e-3, atol=1e-3)


@pytest.mark.gpu
@pytest.mark.parametrize("N,K", [(64, 128), (128, 128)])
def test_probe_a_operand_copied_to_tmem(N, K):
    """tcgen05.cp.128x256b of a SW128 K-major A tile (the MMA's own smem
    descriptor) gives the TS-MMA A layout: same product as the SS MMA."""
    import torch

    lib = _lib()
    torch.manual_seed(2)
    A = torch.randn(128, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    D1 = torch.zeros(128, N, device="cuda")
    D2 = torch.zeros(128, N, device="cuda")
    assert lib.probe_ss_tmem_a(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()), N, K,
                               ctypes.c_void_p(D1.data_ptr()), 0) == 0, lib.probe_last_error()
    assert lib.probe_ss_tmem_a(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()), N, K,
                               ctypes.c_void_p(D2.data_ptr()), 1) == 0, lib.probe_last_error()
    assert torch.equal(D1, D2)
