"""Host-side check of the glibc-expf restatement used by the fp32-exact
kernels (paper_2603_13289_b200/csrc/glibc_expf.h): compiled for the host, it
must equal this host's libm expf bit for bit (every 61st float, ~70M inputs).
The GPU test (tests/test_gpu_kernels.py) checks the device build the same way."""
import ctypes as C
import os
import subprocess
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = r'''
#include <math.h>
#include <stdint.h>
#include <string.h>
#include "glibc_expf.h"
extern "C" uint64_t check(uint32_t stride, uint32_t* first_bad) {
  uint64_t bad = 0;
  for (uint64_t u = 0; u <= 0xffffffffull; u += stride) {
    float x; uint32_t b = (uint32_t)u; memcpy(&x, &b, 4);
    if (isnan(x)) continue;
    float a = rk::glibc_expf(x), r = expf(x);
    uint32_t ua, ur; memcpy(&ua, &a, 4); memcpy(&ur, &r, 4);
    if (ua != ur) { if (!bad) *first_bad = b; ++bad; }
  }
  return bad;
}
'''


def test_glibc_expf_restatement_matches_host_libm():
    with tempfile.TemporaryDirectory() as d:
        cpp = os.path.join(d, "e.cpp")
        open(cpp, "w").write(SRC)
        so = os.path.join(d, "e.so")
        subprocess.run(["g++", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-I",
                        os.path.join(ROOT, "paper_2603_13289_b200", "csrc"), cpp, "-o", so, "-lm"], check=True)
        lib = C.CDLL(so)
        lib.check.restype = C.c_uint64
        lib.check.argtypes = [C.c_uint32, C.POINTER(C.c_uint32)]
        first = C.c_uint32(0)
        bad = lib.check(61, C.byref(first))
        assert bad == 0, f"{bad} mismatches vs libm expf, first input bits {first.value:#010x}"
