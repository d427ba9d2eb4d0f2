"""Test-only alias package: ``sliceplan.<module>`` -> this repo's modules.

Lets the reference's own test files (/root/reference/pkg/tests, read in place,
never copied) import this package under the reference's module names, so
``tests/test_reference_suite.py`` can run them against both implementations
and compare the outcomes.  Module map (reference src/sliceplan/ -> here):

    pipeline.py                                   -> schedule.py
    perf_model.py                                 -> costs.py
    rate_solver.py, memory_assigner.py,
    token_assigner.py, _piecewise.py              -> planner.py
    slicing_kernel.py                             -> sliced.py
    testbeds.py                                   -> desk_profiles.py
    errors.py                                     -> errors.py
"""

import sys

from paper_2411_15715_b200 import costs, desk_profiles, errors, planner, schedule, sliced

for _name, _mod in {"errors": errors, "memory_assigner": planner, "rate_solver": planner,
                    "token_assigner": planner, "_piecewise": planner, "perf_model": costs,
                    "pipeline": schedule, "slicing_kernel": sliced, "testbeds": desk_profiles}.items():
    sys.modules[f"{__name__}.{_name}"] = _mod
