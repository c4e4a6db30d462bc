"""The C++ host API (include/spmmkit, the reference's signatures over the C ABI).

CPU: the headers compile (g++ -std=c++20) and the test program links against
libdaspmm.so. GPU: the program runs the reference-style suite on the device.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_spmmkit_b200.cpp")
PKG = os.path.join(ROOT, "paper_2202_08556_b200")
BIN = os.path.join(PKG, "_build", "test_spmmkit_b200")


def _build():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    if os.path.exists(BIN) and os.path.getmtime(BIN) >= max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(PKG, "libdaspmm.so")),
            *[os.path.getmtime(os.path.join(ROOT, "include", "spmmkit", f))
              for f in os.listdir(os.path.join(ROOT, "include", "spmmkit"))]):
        return BIN
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", BIN,
           "-L", PKG, "-ldaspmm", f"-Wl,-rpath,{PKG}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return BIN


def test_cpp_api_compiles_and_links():
    from paper_2202_08556_b200 import build

    build.build()
    _build()


@pytest.mark.gpu
def test_cpp_api_suite_on_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    b = _build()
    r = subprocess.run([b], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
