"""The user-facing examples run end to end on the GPU (small sizes): sedimentation onto a floor and
the moving-lid piston (NEXT rows f1, f2)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("script,args", [("sedimentation.py", ["2000", "5"]), ("piston.py", ["1500", "5"])])
def test_example_runs(script, args):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "examples", script)] + args, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip(), "the example prints its progress"
