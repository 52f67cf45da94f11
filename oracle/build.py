"""Build the oracle's C restatements (TEST INFRASTRUCTURE ONLY) into
oracle/_build/.  The reference itself is pure Python (no C sources to
compile into oracle/_ref), so only the restatements are native here."""

from __future__ import annotations

import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "_build"


def build() -> Path:
    OUT.mkdir(exist_ok=True)
    lib = OUT / "liboracle_arena.so"
    src = HERE / "arena_oracle.c"
    if src.exists() and (not lib.exists() or lib.stat().st_mtime < src.stat().st_mtime):
        subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-o", str(lib), str(src)], check=True)
    return lib


if __name__ == "__main__":
    print(build())
