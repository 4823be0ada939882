"""pytest plugin for the reference's test_smoke.py run through the `pafft`
alias: the one intended behaviour change is marked xfail (strict).  The
reference rejects radix 3 (`pafft.Plan(3, [9])` raises, test_smoke.py:70,
core.hpp:14-19); this build supports radix 3 and 5 (BASELINE configs 2 and 5),
so test_plan_properties_and_errors is expected to fail on exactly that line."""
import pytest

INTENDED = {
    "test_plan_properties_and_errors": "radix 3 is supported here (BASELINE config 2); the reference rejects it",
}


def pytest_collection_modifyitems(config, items):
    for item in items:
        why = INTENDED.get(item.name)
        if why:
            item.add_marker(pytest.mark.xfail(reason=why, strict=True, raises=pytest.fail.Exception))
