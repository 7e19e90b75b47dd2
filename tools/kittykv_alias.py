"""pytest plugin: run the reference's own tests (kittykv's pkg/tests) against
this package -- `import kittykv` resolves to paper_2511_18643_b200 -- and mark
the cases that exercise parts of the reference outside the device hot path as
expected failures, with the reason (SURVEY.md §2 scope column)."""
import sys

import pytest

import paper_2511_18643_b200 as _kb

OUT_OF_SCOPE = {}


def pytest_configure(config):
    sys.modules["kittykv"] = _kb


def pytest_collection_modifyitems(config, items):
    for item in items:
        nid = item.nodeid.split("/")[-1]
        for key, why in OUT_OF_SCOPE.items():
            if nid.startswith(key):
                item.add_marker(pytest.mark.xfail(reason=why, strict=False))
