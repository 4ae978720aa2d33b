"""CPU checks of the C ABI: the library loads and exports every symbol that
include/stokescol.h declares (no compute calls: there is no GPU here), and
the host-only partition helper behaves."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1909_06623_b200 import _lib, plan_partition

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "stokescol.h")


def _declared():
    txt = open(HDR).read()
    pat = r"^(?:int|void|int64_t|const char)\s*\*?\s*(sc_\w+)\s*\("
    return sorted(set(re.findall(pat, txt, flags=re.M)))


def test_header_declarations_match_binding():
    assert _declared() == sorted(_lib.EXPORTS)


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in _declared():
        assert re.search(rf"\bT {name}\b", out), name
    assert lib.sc_version() == 10000


def test_no_device_context_without_gpu():
    lib = _lib.load()
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    h = ctypes.c_void_p()
    rc = lib.sc_create(ctypes.byref(h), 0, None)
    assert rc < 0  # fails loudly: no silent CPU fallback


@pytest.mark.parametrize("n,world", [(262144, 1), (262144, 2), (262144, 8), (8192, 4), (1000, 3), (512, 8), (1, 2)])
def test_partition_covers_rows_once(n, world):
    parts = [plan_partition(n, world, r) for r in range(world)]
    npad = parts[0]["npad"]
    assert npad % 512 == 0 and npad >= n and npad - n < 512
    covered = []
    for p in parts:
        assert p["row_lo"] % 256 == 0 and p["row_hi"] % 256 == 0
        assert p["chunk_lo"] == p["row_lo"] // 256 and p["chunk_hi"] == p["row_hi"] // 256
        covered += list(range(p["row_lo"], p["row_hi"]))
        assert p["nsplit"] == parts[0]["nsplit"]  # nsplit independent of the rank
    assert covered == list(range(npad))
    # nsplit depends on N only (bitwise P-invariance of the RPY sums)
    assert parts[0]["nsplit"] == plan_partition(n, 1, 0)["nsplit"]


def _build_c_demo(out):
    lib_dir = os.path.join(ROOT, "paper_1909_06623_b200")
    _lib.load()  # (builds the library if missing)
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "c_api_demo.c"), "-L", lib_dir, "-lstokescol",
           f"-Wl,-rpath,{lib_dir}", "-lm", "-o", out]
    return subprocess.run(cmd, capture_output=True, text=True)


def test_c_demo_compiles_against_the_header(tmp_path):
    """The boundary is a plain C ABI: examples/c_api_demo.c builds with gcc (C, no C++) against
    include/stokescol.h and links libstokescol.so."""
    r = _build_c_demo(str(tmp_path / "c_api_demo"))
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_c_demo_runs(tmp_path):
    exe = str(tmp_path / "c_api_demo")
    assert _build_c_demo(exe).returncode == 0
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "c_api_demo: ok" in r.stdout, r.stdout + r.stderr
