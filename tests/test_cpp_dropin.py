"""The C++ drop-in API (include/ngemm) built and run as a client would use it:
  * our own suite tests/cpp/test_dropin.cpp, and
  * the reference's OWN unit-test sources (test_gemm/test_layout/test_matrix/test_lanes.cpp)
    compiled against our headers (built where /root/reference exists; the binary travels
    to the GPU box).  Every case passes on the GPU, including the i16 ones."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")
BUILD = os.path.join(CPP, "build")


def _make(target):
    subprocess.run(["make", "-s", "-C", CPP, target], check=True, capture_output=True, text=True)


def test_dropin_headers_compile():
    _make("dropin")
    assert os.path.exists(os.path.join(BUILD, "dropin_tests"))


def test_reference_suites_compile_against_dropin_headers():
    if not os.path.exists("/root/reference/proj/tests/test_gemm.cpp"):
        pytest.skip("reference sources not present (only in the build container)")
    _make("conformance")
    assert os.path.exists(os.path.join(BUILD, "ref_conformance"))


def test_reference_suites_host_cases_pass_without_gpu():
    """Host-only cases (lanes, layout, matrix, oracles) pass anywhere; GEMM cases need the GPU
    and must FAIL loudly here (CudaError), never silently run on the CPU."""
    import torch
    exe = os.path.join(BUILD, "ref_conformance")
    if not os.path.exists(exe):
        pytest.skip("ref_conformance not built")
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu test")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600).stdout
    for line in out.splitlines():
        if line.startswith("  FAILED") and "unexpected exception" in line:
            assert "CUDA" in line or "cuda" in line, line
    assert "55 test cases" in out


@pytest.mark.gpu
def test_dropin_suite_on_gpu(cuda):
    _make("dropin")
    r = subprocess.run([os.path.join(BUILD, "dropin_tests")], capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:]


@pytest.mark.gpu
def test_reference_suites_on_gpu(cuda):
    exe = os.path.join(BUILD, "ref_conformance")
    if not os.path.exists(exe):
        pytest.fail("tests/cpp/build/ref_conformance missing: build it where the reference exists "
                    "(make -C tests/cpp conformance) before shipping the snapshot")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:]
    assert "55 test cases, 0 failed" in r.stdout
