# Offline install of the unmodified reference (kittykv) into baseline/_ref for the
# bench's reference arm, and a copy of its own tests into baseline/_ref_tests for
# tools/run_reference_suite.py.  Both directories are git-ignored (not sources of
# this repo) but travel to the GPU box with gpurun.  Run in the build container.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/kittykv_src && cp -r /root/reference/pkg /tmp/kittykv_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref --upgrade /tmp/kittykv_src
rm -rf baseline/_ref_tests && mkdir -p baseline/_ref_tests && cp /root/reference/pkg/tests/test_pages.py \
    /root/reference/pkg/tests/test_cache.py /root/reference/pkg/tests/test_quant.py \
    /root/reference/pkg/tests/test_analysis.py baseline/_ref_tests/
