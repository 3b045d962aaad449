"""GPU pins of the raw-PTX building blocks (tests/cuda/umma_probe.cu) against
torch matmuls: TMA SW128 loads, UMMA K-major / MN-major smem descriptors,
A-operand from TMEM, manual swizzled smem writes, tcgen05.ld/st/commit."""
import ctypes
import os

import pytest
import torch

pytestmark = pytest.mark.gpu

SO = os.path.join(os.path.dirname(__file__), "cuda", "libumma_probe.so")


@pytest.fixture(scope="module")
def probe(cuda_ok):
    lib = ctypes.CDLL(SO)
    lib.probe_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    lib.probe_run.restype = ctypes.c_int
    return lib


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_umma_modes(probe, mode):
    g = torch.Generator(device="cpu").manual_seed(mode)
    a = torch.randn(128, 128, generator=g).to(torch.bfloat16).cuda()
    b = torch.randn(128, 128, generator=g).to(torch.bfloat16).cuda()
    d = torch.full((128, 128), float("nan"), device="cuda")
    rc = probe.probe_run(mode, a.data_ptr(), b.data_ptr(), d.data_ptr())
    assert rc == 0, rc
    af, bf = a.double().cpu(), b.double().cpu()
    if mode == 0:
        ref = af @ bf.T      # D[m][n] = sum_k A[m][k] B[n][k]
    elif mode == 1:
        ref = af @ bf        # D[m][n] = sum_k P[m][k] V[k][n]
    else:
        ref = af.T @ bf      # D[m][n] = sum_k X[k][m] Y[k][n]
    err = (d.double().cpu() - ref).abs().max().item()
    assert err < 1e-3, f"mode {mode}: max abs err {err}"
