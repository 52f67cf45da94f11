"""The product path fails loudly when libdvla_b200.so is absent.

There is no CPU fallback (DESIGN.md §1 "Boundary"): the native binding
raises ImportError on import, and compute entry points (which import it
lazily so the host-side types stay importable without a GPU) raise the same
error on their first call rather than route through `oracle/` or numpy.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("stmt", [
    "import paper_2605_13276_b200._lib",
    "import numpy as np; from paper_2605_13276_b200 import grpo; "
    "grpo.compute_advantages(np.array([1.0, 0.0, 2.0, 3.0]), 1e-8)",
])
def test_missing_library_raises_import_error(stmt, tmp_path):
    env = dict(os.environ, DVLA_B200_LIB=str(tmp_path / "libdvla_b200.so"))
    code = (f"try:\n"
            f"    {stmt}\n"
            f"except ImportError as e:\n"
            f"    assert 'no CPU fallback' in str(e), e\n"
            f"    print('raised')\n"
            f"else:\n"
            f"    raise SystemExit('ran without the native library')\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "raised" in r.stdout
