"""The C-ABI from plain C (no Python, no torch): the header compiles as C,
and on a GPU a C program calls dvla_token_loss_fwd_bwd and checks it
against its own scalar restatement of the reference loss."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2605_13276_b200")
SRC = os.path.join(ROOT, "tests", "c_abi", "token_loss_c.c")
CUDA = "/usr/local/cuda"


def _gcc(*extra):
    return ["gcc", "-std=c11", "-O1", "-Wall", "-Werror", f"-I{ROOT}/include",
            f"-I{CUDA}/include", *extra]


def test_header_and_caller_compile_as_c():
    res = subprocess.run(_gcc("-fsyntax-only", SRC), capture_output=True, text=True)
    assert res.returncode == 0, res.stderr


@pytest.mark.gpu
def test_plain_c_caller_runs_the_token_loss(tmp_path):
    exe = str(tmp_path / "token_loss_c")
    res = subprocess.run(_gcc(SRC, "-o", exe, f"-L{PKG}", "-ldvla_b200", f"-Wl,-rpath,{PKG}",
                              f"-L{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{CUDA}/lib64", "-lm"),
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    run = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "C_ABI_OK" in run.stdout
