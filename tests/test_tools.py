"""The tools/ scripts (sweeps, A/B, ncu drivers, sanitizer, microbenchmarks)
run only on a GPU box; here they must at least compile, and the ones with a
CLI must parse their arguments (so they cannot rot silently)."""
import glob
import os
import py_compile
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_tools_compile():
    files = sorted(glob.glob(os.path.join(ROOT, "tools", "*.py")))
    assert files
    for f in files:
        py_compile.compile(f, doraise=True)


def test_sanitize_cases_listed():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize.py"), "list"], capture_output=True,
                       text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    cases = r.stdout.split()
    for c in ("cta_batch32", "grid_frontier", "groups", "part_rounds", "peer_loopback"):
        assert c in cases


def test_sweep_cli_help():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sweep.py"), "--help"], capture_output=True,
                       text=True, timeout=120, cwd=ROOT)
    assert r.returncode == 0 and "WORKLOAD" in r.stdout
