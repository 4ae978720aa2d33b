"""The oracle and the product share no code (task rule): the package never imports the oracle,
the oracle never includes product headers or imports the package (except the seeded input
generator, which holds no arithmetic of the method), and the product fails loudly without its
CUDA library instead of falling back to CPU code."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1909_06623_b200")
ORC = os.path.join(ROOT, "oracle")


def _files(d, exts):
    for base, _, names in os.walk(d):
        for n in names:
            if n.endswith(exts):
                yield os.path.join(base, n)


def test_product_never_imports_the_oracle():
    for f in _files(PKG, (".py", ".cu", ".cuh", ".h")):
        txt = open(f, encoding="utf-8").read()
        assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, flags=re.M), f
        assert "liboracle" not in txt and "oracle.h" not in txt, f


def test_oracle_includes_no_product_code():
    for f in _files(ORC, (".c", ".h", ".py")):
        txt = open(f, encoding="utf-8").read()
        assert "stokescol.h" not in txt and "sc_internal.h" not in txt and "csrc" not in txt, f
        assert "libstokescol" not in txt, f
        for m in re.finditer(r"^\s*(?:import|from)\s+(paper_1909_06623_b200[\w.]*)", txt, flags=re.M):
            assert m.group(1) == "paper_1909_06623_b200.synthetic", (f, m.group(1))


def test_synthetic_inputs_hold_no_method_arithmetic():
    """The only shared module draws inputs: no RPY, contact, D or BBPGD arithmetic in it."""
    txt = open(os.path.join(PKG, "synthetic.py"), encoding="utf-8").read()
    for word in ("rsqrt", "mobility(", "bbpgd", "apply_D", "gap ="):
        assert word not in txt, word


def test_binding_has_no_cpu_fallback():
    txt = open(os.path.join(PKG, "_lib.py"), encoding="utf-8").read()
    assert "raise RuntimeError" in txt  # missing library -> loud error
    api = open(os.path.join(PKG, "api.py"), encoding="utf-8").read()
    assert "numpy.linalg" not in api and "np.linalg" not in api
