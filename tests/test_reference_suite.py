"""The reference's own test suite, run against this package (drop-in check).

``/root/reference/pkg/tests`` is executed twice in subprocesses, read in place
(nothing is copied into this repo):

1. against the reference package itself (``/root/reference/pkg/src``);
2. against this package through ``tests/refshim/sliceplan`` (an alias package
   mapping the reference's module names onto ours).

Every test id must end with the same outcome in both runs.  A test that fails
must fail the same way in both, with the same assertion message.  The
reference's ``test_acceptance.py::test_criterion_4`` fails on the reference
itself, and ours reproduces its numbers digit for digit.

Not run against this package:

* ``test_cli.py``: the reference CLI is out of scope.
* The fp64 recombination tests (``TestRecombination`` and acceptance
  criterion 5).  They call ``mlp_forward_sliced`` and expect <= 1e-12 against
  an fp64 dense forward.  Our forward runs the GG / CG blocks on the GPU with
  no CPU fallback, in fp32 / bf16.  Its numerics are tested on the GPU in
  ``test_sliced_api.py`` / ``test_gpu_parity.py`` at the north star's
  tolerance (fp32 <= 1e-5, bf16 <= 1e-2 max relative error).

This needs the reference checkout, so it is skipped where that is absent
(on the GPU box).
"""

from __future__ import annotations

import os
import subprocess
import sys
import xml.etree.ElementTree as ET
from pathlib import Path

import pytest

REF_TESTS = Path("/root/reference/pkg/tests")
REF_SRC = Path("/root/reference/pkg/src")
REPO = Path(__file__).resolve().parents[1]
SHIM = Path(__file__).resolve().parent / "refshim"

NOT_PORTED = "not TestRecombination and not test_criterion_5_slicing_recombination"

pytestmark = pytest.mark.skipif(not (REF_TESTS.is_dir() and REF_SRC.is_dir()),
                                reason="reference checkout not present")


def _run_suite(tmp: Path, pythonpath: str, tag: str) -> dict[str, tuple[str, str]]:
    """Run the reference tests; return {test id: (outcome, first message line)}."""
    work = tmp / tag
    work.mkdir()
    (work / "pytest.ini").write_text("[pytest]\n")
    xml = work / "junit.xml"
    env = dict(os.environ, PYTHONPATH=pythonpath, PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-c", str(work / "pytest.ini"),
           "--rootdir", str(work), f"--junitxml={xml}", "-k", NOT_PORTED,
           "--ignore", str(REF_TESTS / "test_cli.py"), str(REF_TESTS)]
    proc = subprocess.run(cmd, cwd=work, env=env, capture_output=True, text=True, timeout=900)
    assert xml.exists(), proc.stdout[-3000:] + proc.stderr[-3000:]
    out = {}
    for case in ET.parse(xml).getroot().iter("testcase"):
        tid = f"{case.get('classname')}::{case.get('name')}"
        outcome, msg = "passed", ""
        for kind in ("failure", "error", "skipped"):
            el = case.find(kind)
            if el is not None:
                outcome = kind
                msg = (el.get("message") or "").splitlines()[0] if el.get("message") else ""
                break
        out[tid] = (outcome, msg)
    return out


def test_reference_suite_same_outcomes(tmp_path):
    ref = _run_suite(tmp_path, str(REF_SRC), "reference")
    ours = _run_suite(tmp_path, os.pathsep.join([str(SHIM), str(REPO)]), "ours")
    assert len(ref) > 100, f"only {len(ref)} reference tests collected"
    assert set(ours) == set(ref), sorted(set(ours) ^ set(ref))[:10]
    diff = {t: (ref[t], ours[t]) for t in ref if ref[t] != ours[t]}
    assert not diff, "\n".join(f"{t}: reference {r} / ours {o}" for t, (r, o) in sorted(diff.items())[:10])
    n_pass = sum(o == "passed" for o, _ in ours.values())
    # the reference's only failing test must stay the known criterion-4 one (identical detail on both sides)
    failing = sorted(t for t, (o, _) in ours.items() if o != "passed")
    assert all("criterion_4" in t for t in failing), failing
    assert n_pass >= len(ours) - 1
