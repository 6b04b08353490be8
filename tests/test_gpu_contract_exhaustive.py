"""Exhaustive bitwise comparison of the contract math, oracle vs GPU (SURVEY
8c-2 "Contract math itself"): for exp2, log2(1-p), rcp and rsqrt over every
fp32 input of their domain, lowbias32 over all 2^32 inputs, and atan2-in-turns
over 2^30 hashed finite pairs, an order-independent 64-bit checksum of the
output bits computed by the oracle's C functions (host threads) equals the
one computed by the product's device functions (tests/contract_selftest.cu,
including paper_2306_05051_b200/csrc/glint_device.cuh)."""
import ctypes as C
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.fixture(scope="module")
def selftest():
    out = os.path.join(ROOT, "tests", "libcontract_selftest.so")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-fmad=false", "-prec-div=true",
           "-prec-sqrt=true", "-ftz=false", "-Xcompiler", "-fPIC", "-shared", "-o", out,
           os.path.join(ROOT, "tests", "contract_selftest.cu")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    L = C.CDLL(out)
    L.contract_checksum.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]
    L.contract_checksum.restype = C.c_int
    return L


@pytest.mark.timeout(900)
@pytest.mark.parametrize("fn,name,hi", [(0, "exp2", 1 << 32), (1, "log2_1mp", 1 << 32), (2, "rcp", 1 << 32),
                                        (3, "rsqrt", 1 << 32), (5, "lowbias32", 1 << 32), (4, "atan2_turns", 1 << 30)])
def test_contract_function_bit_equal_on_every_input(selftest, fn, name, hi):
    import oracle
    g = C.c_uint64(0)
    assert selftest.contract_checksum(fn, 0, hi, C.byref(g)) == 0
    o = oracle.contract_checksum(fn, 0, hi)
    assert g.value == o, (name, hex(g.value), hex(o))
