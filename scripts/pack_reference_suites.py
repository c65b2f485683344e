#!/usr/bin/env python
"""Pack the reference's own hot-path test suites into a test fixture.

Run in the authoring container (the GPU box has no /root/reference):

    python scripts/pack_reference_suites.py

Writes tests/golden/reference_suites.tar.gz: the reference's pkg/tests files
for the path this package replaces (core, occupancy, grid,
batched, render) plus their conftest/helpers, byte for byte.  They are test
infrastructure -- tests/test_reference_suites.py runs them, unmodified,
against this package with `gridfield` aliased to it (drop-in proof).
"""

import io
import os
import tarfile
from pathlib import Path

SRC = Path(os.environ.get("GRIDFIELD_REFERENCE_TESTS", "/root/reference/pkg/tests"))
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "reference_suites.tar.gz"
FILES = ["conftest.py", "helpers.py", "test_core.py", "test_occupancy.py", "test_grid.py", "test_batched.py",
         "test_render.py", "test_mlp.py"]


def main():
    with tarfile.open(OUT, "w:gz") as tar:
        for f in FILES:
            data = (SRC / f).read_bytes()
            info = tarfile.TarInfo(f"reference_tests/{f}")
            info.size = len(data)
            info.mtime = 0
            tar.addfile(info, io.BytesIO(data))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(FILES)} files)")


if __name__ == "__main__":
    main()
