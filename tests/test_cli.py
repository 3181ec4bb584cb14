"""The `ngemm` CLI (tools/ngemm_cli.cpp; SPEC.md:456-529 cmd_pack / cmd_gemm / cmd_bench, plus tune)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "bin", "ngemm")


def run(*args, check=True):
    r = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)
    if check and r.returncode != 0:
        raise AssertionError(f"ngemm {' '.join(args)} failed: {r.stderr}")
    return r


@pytest.fixture(scope="module", autouse=True)
def built():
    subprocess.run(["make", "-s", "-C", ROOT, "bin/ngemm"], check=True, capture_output=True)


def _read_ngmm(path):
    raw = open(path, "rb").read()
    assert raw[:4] == b"NGMM"
    kind = raw[8]
    rows = int.from_bytes(raw[9:17], "little")
    cols = int.from_bytes(raw[17:25], "little")
    dt = {0: np.uint8, 1: np.int8, 2: np.int16, 3: np.int32}[kind]
    return np.frombuffer(raw[25:], dtype=dt).reshape(rows, cols)


def test_cli_host_commands(tmp_path, oracle):
    a, b, w, c = (str(tmp_path / x) for x in ("a.ngmm", "b.ngmm", "w.ngpt", "c.ngmm"))
    run("rand", "--kind", "u8", "--rows", "37", "--cols", "101", "--seed", "5", "--out", a)
    run("rand", "--kind", "i8", "--rows", "20", "--cols", "101", "--seed", "6", "--out", b)
    # rand is the reference's mat_random (matrix.hpp:131-143): same stream as the oracle
    assert (_read_ngmm(a) == oracle.mat_random_u8(37, 101, 5)).all()
    out = run("pack", "--in", a, "--out", w, "--isa", "v256", "--tile", "8,4,12", "--perm", "nkm").stdout
    assert "m_pad=40 k_pad=108" in out and os.path.getsize(w) == 25 + 40 * 108 + 57
    run("gemm", "--a", a, "--b", b, "--variant", "ref", "--mode", "sat", "--out", c)
    assert (_read_ngmm(c) == oracle.gemm(_read_ngmm(a), _read_ngmm(b), 0)).all()
    # spec negatives: packed file to variant ref is a pairing error; i32 cannot be packed
    assert run("gemm", "--packed", w, "--b", b, "--variant", "ref", check=False).returncode != 0
    i32 = str(tmp_path / "i.ngmm")
    run("rand", "--kind", "i32", "--rows", "2", "--cols", "2", "--lo", "0", "--hi", "3", "--out", i32)
    assert run("pack", "--in", i32, "--out", w, check=False).returncode != 0


def test_cli_gpu_commands_fail_loudly_without_gpu(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    a, b = str(tmp_path / "a.ngmm"), str(tmp_path / "b.ngmm")
    run("rand", "--kind", "u8", "--rows", "4", "--cols", "8", "--out", a)
    run("rand", "--kind", "i8", "--rows", "4", "--cols", "8", "--out", b)
    r = run("gemm", "--a", a, "--b", b, "--variant", "conventional", check=False)
    assert r.returncode != 0 and "CUDA" in r.stderr


@pytest.mark.gpu
def test_cli_gemm_variants_identical_files(cuda, tmp_path):
    a, b, w = (str(tmp_path / x) for x in ("a.ngmm", "b.ngmm", "w.ngpt"))
    run("rand", "--kind", "u8", "--rows", "300", "--cols", "777", "--seed", "1", "--out", a)
    run("rand", "--kind", "i8", "--rows", "129", "--cols", "777", "--seed", "2", "--out", b)
    run("pack", "--in", a, "--out", w, "--tile", "32,64,64", "--perm", "kmn")
    for mode in ("exact", "sat"):
        outs = {}
        for v in ("ref", "conventional", "ngemm"):
            o = str(tmp_path / f"c_{v}_{mode}.ngmm")
            src = ("--packed", w) if v == "ngemm" else ("--a", a)
            run("gemm", *src, "--b", b, "--variant", v, "--mode", mode, "--out", o)
            outs[v] = open(o, "rb").read()
        assert outs["ref"] == outs["conventional"] == outs["ngemm"], mode  # byte-for-byte (SPEC cmd_gemm)


@pytest.mark.gpu
def test_cli_bench_and_tune(cuda, tmp_path):
    csv = str(tmp_path / "bench.csv")
    out = run("bench", "--sizes", "64x64x128,256x256x1024", "--repeats", "3", "--warmup", "1", "--out", csv).stdout
    lines = open(csv).read().splitlines()
    assert lines[0] == "m,n,k,kind,isa,variant,median_ns,min_ns,trials,checksum"
    rows = [l.split(",") for l in lines[1:] if not l.startswith("#")]
    assert len(rows) == 4 and {r[5] for r in rows} == {"conventional", "ngemm"}
    assert rows[0][9] == rows[1][9]  # identical checksum across variants
    assert "geomean" in out
    store = str(tmp_path / "tune.txt")
    out = run("tune", "--sizes", "512x512x512,8x4096x1024", "--repeats", "3", "--warmup", "1", "--store", store).stdout
    assert out.count("kernel=") == 2 and len(open(store).read().splitlines()) == 2
