"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol that
include/ngemm_cuda.h declares, validates before launching (reference error mapping), and
fails loudly — never falls back to the CPU — when no GPU is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1910_00178_b200 import _lib, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "ngemm_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ngemm_cuda_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(_lib.EXPORTS) == declared


def test_abi_version_and_status_names():
    L = _lib.load()
    assert L.ngemm_cuda_abi_version() == 1
    names = [L.ngemm_cuda_status_name(i).decode() for i in range(9)]
    assert names == ["ok", "ShapeError", "UnsupportedError", "ConfigError", "RangeError", "CorruptionError",
                     "IndexError", "CudaError", "TuneError"]


def test_kernel_pick_policy():
    assert api.pick_kernel(1, 768, 768, api.SatMode.WIDENING_EXACT) == "skinny"
    assert api.pick_kernel(16, 4096, 1024, api.SatMode.HARDWARE_SATURATING) == "skinny"
    assert api.pick_kernel(1024, 1024, 1024, api.SatMode.WIDENING_EXACT) == "tcgen05"
    # saturating: the tensor-core hybrid from M >= 256 and 1e9 MACs, the CUDA-core kernel below
    assert api.pick_kernel(1024, 1024, 1024, api.SatMode.HARDWARE_SATURATING) == "sat_hybrid"
    assert api.pick_kernel(512, 1024, 1024, api.SatMode.HARDWARE_SATURATING) == "simt"
    assert api.pick_kernel(128, 4096, 4096, api.SatMode.HARDWARE_SATURATING) == "simt"
    assert api.pick_kernel(17, 64, 64, api.SatMode.WIDENING_EXACT) == "tcgen05"


def test_shard_rows():
    assert api.shard_rows(16384, 8, 128) == [0, 2048, 4096, 6144, 8192, 10240, 12288, 14336, 16384]
    assert api.shard_rows(1000, 4, 128) == [0, 256, 512, 768, 1000]
    assert api.shard_rows(100, 4, 128) == [0, 100, 100, 100, 100]
    rs = api.shard_rows(16385, 8, 128)
    assert rs[0] == 0 and rs[-1] == 16385 and all(r % 128 == 0 for r in rs[:-1])


def test_packed_validate_maps_config_errors():
    L = _lib.load()
    good = _lib.PackedMeta(32, 4, 8, 8, 1, 4, 0, 5, 5, 8, 8)
    assert L.ngemm_cuda_packed_validate(C.byref(good)) == _lib.OK
    for bad in (_lib.PackedMeta(32, 4, 8, 7, 1, 4, 0, 5, 5, 7, 8),     # tm not multiple of v
                _lib.PackedMeta(32, 4, 8, 8, 1, 5, 0, 5, 5, 8, 5),     # tk not multiple of h
                _lib.PackedMeta(32, 4, 8, 8, 0, 4, 0, 5, 5, 8, 8),     # tn < 1
                _lib.PackedMeta(32, 2, 16, 8, 1, 4, 0, 5, 5, 8, 8)):   # 16-bit shape on the u8 path
        assert L.ngemm_cuda_packed_validate(C.byref(bad)) == _lib.ERR_CONFIG
    wrong_pad = _lib.PackedMeta(32, 4, 8, 8, 1, 4, 0, 5, 5, 16, 8)
    assert L.ngemm_cuda_packed_validate(C.byref(wrong_pad)) == _lib.ERR_SHAPE


def test_validation_precedes_device_use():
    # errors are reported before any launch, like the reference throws before dispatch
    L = _lib.load()
    buf = (C.c_uint8 * 64)()
    assert L.ngemm_cuda_gemm_u8i8(buf, 4, buf, 4, buf, 4, 0, 4, 4, 1, None) == _lib.ERR_SHAPE
    assert L.ngemm_cuda_gemm_u8i8(buf, 3, buf, 4, buf, 4, 4, 4, 4, 1, None) == _lib.ERR_SHAPE
    assert L.ngemm_cuda_gemm_u8i8(buf, 4, buf, 4, buf, 4, 4, 4, 4, 7, None) == _lib.ERR_CONFIG
    # strided batch: C slices may not overlap, operand strides must cover one operand
    B = L.ngemm_cuda_gemm_u8i8_strided_batched
    assert B(buf, 4, 16, buf, 4, 16, buf, 4, 15, 2, 4, 4, 4, 1, None) == _lib.ERR_SHAPE
    assert B(buf, 4, 8, buf, 4, 16, buf, 4, 16, 2, 4, 4, 4, 1, None) == _lib.ERR_SHAPE
    assert B(buf, 4, 16, buf, 4, 16, buf, 4, 16, -1, 4, 4, 4, 1, None) == _lib.ERR_SHAPE
    assert B(buf, 4, 16, buf, 4, 16, buf, 4, 16, 0, 4, 4, 4, 1, None) == _lib.OK  # empty batch: no-op


def test_api_engine_and_kind_errors():
    a = np.zeros((4, 8), np.uint8)
    b = np.zeros((4, 8), np.int8)
    with pytest.raises(api.UnsupportedError):
        api.gemm_conventional(a, b, api.kernel_shape(256), api.SatMode.WIDENING_EXACT, api.Engine.NATIVE)
    with pytest.raises(api.UnsupportedError):
        api.gemm_conventional(a, b.view(np.uint8), api.kernel_shape(256), api.SatMode.WIDENING_EXACT)
    with pytest.raises(api.ShapeError):
        api.gemm_conventional(a, np.zeros((4, 9), np.int8), api.kernel_shape(256), api.SatMode.WIDENING_EXACT)
    p = api.pack_weights(a, api.kernel_shape(256), api.TileConfig(8, 1, 4))
    with pytest.raises(api.ShapeError):
        api.gemm_ngemm(p, np.zeros((4, 9), np.int8), api.SatMode.WIDENING_EXACT)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    a = np.ones((4, 8), np.uint8)
    b = np.ones((4, 8), np.int8)
    with pytest.raises(api.CudaError):
        api.gemm_conventional(a, b, api.kernel_shape(256), api.SatMode.WIDENING_EXACT)


def test_kernel_shape_table():
    # test_layout.cpp:12-22 (8-bit rows)
    assert api.kernel_shape(256) == api.KernelShape(32, 4, 8)
    assert api.kernel_shape(512) == api.KernelShape(64, 4, 16)
    assert api.kernel_shape(128) == api.KernelShape(16, 4, 4)
    assert api.kernel_shape(256, 16) == api.KernelShape(16, 2, 8)
    with pytest.raises(api.UnsupportedError):
        api.kernel_shape(256, 32)


def test_host_pack_matches_oracle_and_reference_digests(oracle, golden):
    for c in golden["packs"]:
        a = np.array([[1, 2], [3, 4]], np.uint8) if c["seed"] is None else oracle.mat_random_u8(c["m"], c["k"], c["seed"])
        p = api.pack_weights(a, api.KernelShape(c["w"], c["h"], c["v"]),
                             api.TileConfig(c["tm"], c["tn"], c["tk"], api.Perm(c["perm"])))
        assert p.data.size == c["nbytes"]
        assert oracle.fnv1a(p.data) == c["fnv"]
        assert (api.unpack_weights(p) == a).all()


def test_host_unpack_detects_corruption():
    a = np.arange(25, dtype=np.uint8).reshape(5, 5) + 1
    p = api.pack_weights(a, api.KernelShape(32, 4, 8), api.TileConfig(8, 1, 4))
    p.data[p.elem_offset(7, 0)] = 42
    with pytest.raises(api.CorruptionError):
        api.unpack_weights(p)


def test_pack_rejects_bad_tiles_and_kinds():
    a = np.zeros((4, 4), np.uint8)
    s = api.KernelShape(32, 4, 8)
    for t in (api.TileConfig(7, 1, 4), api.TileConfig(8, 1, 5), api.TileConfig(8, 0, 4)):
        with pytest.raises(api.ConfigError):
            api.pack_weights(a, s, t)
    with pytest.raises(api.UnsupportedError):
        api.pack_weights(np.zeros((4, 4), np.int32), s, api.TileConfig(8, 1, 4))


def test_tune_store_round_trip_and_malformed(tmp_path):
    # the store is host-side (no GPU needed): append-only lines, last record for a shape wins
    p = tmp_path / "tune.txt"
    p.write_text("# m n k mode kernel cfg splits variant median min trials ts\n"
                 "1024 1024 1024 1 1 3 1 -1 5000 4800 5 1700000000\n"
                 "1024 1024 1024 1 1 2 2 -1 4000 3900 5 1700000001\n"
                 "16 4096 1024 1 3 -1 -1 3 3000 2900 5 1700000002\n")
    api.tune_clear()
    assert api.tune_store_load(str(p)) == 3
    out = tmp_path / "saved.txt"
    api.tune_store_save(str(out))
    lines = [l.split() for l in out.read_text().splitlines()]
    assert len(lines) == 2  # last wins per shape
    assert ["1024", "1024", "1024", "1", "1", "2", "2", "-1"] in [l[:8] for l in lines]
    bad = tmp_path / "bad.txt"
    bad.write_text("1024 1024 x\n")
    with pytest.raises(api.ConfigError):
        api.tune_store_load(str(bad))
    api.tune_clear()


def test_option_table_read_once_and_settable():
    """Experiment knobs: read once from NGEMM_<NAME> (never on the launch path), changed through
    the C-ABI, unknown names rejected with ConfigError, reset re-reads the environment."""
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "from paper_1910_00178_b200 import _lib\n"
        "assert _lib.get_option('TC_CFG') == 3, _lib.get_option('TC_CFG')\n"
        "assert _lib.get_option('NGEMM_TC_CFG') == 3\n"
        "assert _lib.get_option('I16_PATH') == 1\n"
        "assert _lib.get_option('TC_L2HINT') == 7\n"
        "_lib.set_option('TC_CFG', 5); assert _lib.get_option('TC_CFG') == 5\n"
        "with _lib.options(TC_SPLITS=2):\n"
        "    assert _lib.get_option('TC_SPLITS') == 2\n"
        "assert _lib.get_option('TC_SPLITS') == -1\n"
        "_lib.reset_options(); assert _lib.get_option('TC_CFG') == 3\n"
        "assert _lib.get_option('NO_SUCH_KNOB') == -2**31\n"
        "try:\n"
        "    _lib.set_option('NO_SUCH_KNOB', 1)\n"
        "    raise SystemExit('accepted an unknown option')\n"
        "except _lib.ConfigError:\n"
        "    pass\n"
        "print('ok')\n") % ROOT
    env = dict(os.environ, NGEMM_TC_CFG="3", NGEMM_I16_PATH="tcgen05")
    env.pop("NGEMM_TC_L2HINT", None)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stdout + r.stderr
