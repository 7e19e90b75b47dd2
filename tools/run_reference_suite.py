"""Run the reference's own tests/test_pages.py, test_cache.py, test_quant.py and
test_analysis.py (copied
into baseline/_ref_tests by tools/install_reference.sh) against this package on
the GPU: `kittykv` is aliased to paper_2511_18643_b200 (tools/kittykv_alias.py),
out-of-scope cases are xfail with their reason.

    python tools/run_reference_suite.py [pytest args]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.join(ROOT, "baseline", "_ref_tests")

if __name__ == "__main__":
    if not os.path.isdir(TESTS):
        raise SystemExit("baseline/_ref_tests is missing: run tools/install_reference.sh")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "tools")]))
    cmd = [sys.executable, "-m", "pytest", "-p", "kittykv_alias", "-p", "no:cacheprovider", "-rxXs", "-q",
           "--rootdir", TESTS, os.path.join(TESTS, "test_pages.py"), os.path.join(TESTS, "test_cache.py"),
           os.path.join(TESTS, "test_quant.py"), os.path.join(TESTS, "test_analysis.py")] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd, env=env, cwd=TESTS))
