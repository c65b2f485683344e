#!/usr/bin/env python
"""Run the reference's own test files (tests/golden/reference_suites.tar.gz,
packed by scripts/pack_reference_suites.py) against THIS package: the files
are extracted unmodified next to a `gridfield` shim whose modules are this
package's modules, and pytest runs them in a child process.

    python scripts/run_reference_suites.py [--out results.json] [pytest args]

Prints one JSON object: {"passed": [...], "failed": [...], "skipped": [...],
"errors": [...]} keyed by test node id (file::name[param]).
"""

import argparse
import json
import os
import subprocess
import sys
import tarfile
import tempfile
import xml.etree.ElementTree as ET
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
ARCHIVE = ROOT / "tests" / "golden" / "reference_suites.tar.gz"

SHIM = '''"""`gridfield` -> paper_2103_13744_b200 (drop-in alias for the reference's tests)."""
import importlib as _il
import sys as _sys

from paper_2103_13744_b200 import *  # noqa: F401,F403

for _m in ("core", "grid", "batched", "mlp", "occupancy", "render", "scene", "io", "train"):
    _mod = _il.import_module("paper_2103_13744_b200." + _m)
    _sys.modules[__name__ + "." + _m] = _mod
    globals()[_m] = _mod
'''


def run(pytest_args=(), timeout=1800, env_extra=None):
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        with tarfile.open(ARCHIVE) as tar:
            tar.extractall(tmp, filter="data")
        shim = tmp / "shim" / "gridfield"
        shim.mkdir(parents=True)
        (shim / "__init__.py").write_text(SHIM)
        tests = tmp / "reference_tests"
        junit = tmp / "junit.xml"
        env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(tmp / "shim"), str(ROOT), env_pp()]),
                   PYTHONDONTWRITEBYTECODE="1", **(env_extra or {}))
        targets = [str(tests / a) for a in pytest_args if a.endswith(".py")] or [str(tests)]
        extra = [a for a in pytest_args if not a.endswith(".py")]
        cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", str(tests),
               f"--junitxml={junit}", *targets, *extra]
        proc = subprocess.run(cmd, cwd=tests, env=env, capture_output=True, text=True, timeout=timeout)
        res = {"passed": [], "failed": [], "skipped": [], "errors": [], "returncode": proc.returncode,
               "tail": proc.stdout[-3000:] + proc.stderr[-2000:]}
        if junit.exists():
            for tc in ET.parse(junit).getroot().iter("testcase"):
                name = f"{tc.get('file') or tc.get('classname', '').replace('.', '/') + '.py'}::{tc.get('name')}"
                name = name.replace("reference_tests/", "")
                kids = {c.tag: c for c in tc}
                if "failure" in kids:
                    res["failed"].append([name, (kids["failure"].get("message") or "")[:300]])
                elif "error" in kids:
                    res["errors"].append([name, (kids["error"].get("message") or "")[:300]])
                elif "skipped" in kids:
                    res["skipped"].append([name, (kids["skipped"].get("message") or "")[:200]])
                else:
                    res["passed"].append(name)
        return res


def env_pp():
    return os.environ.get("PYTHONPATH", "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    a, rest = ap.parse_known_args()
    res = run(rest)
    s = json.dumps(res, indent=1)
    if a.out:
        Path(a.out).write_text(s)
    print(json.dumps({k: (len(v) if isinstance(v, list) else v) for k, v in res.items() if k != "tail"}))
    for k in ("failed", "errors"):
        for n, m in res[k]:
            print(k.upper(), n, "--", m[:200])


if __name__ == "__main__":
    main()
