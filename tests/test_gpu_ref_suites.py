"""The reference's own test suites, compiled UNCHANGED against the drop-in
headers (include/spike) and libspike_b200.so (oracle/Makefile `suites`;
doctest subset in tests/cpp/doctest; test helpers generate / oracle /
band_ops from the reference sources).  SURVEY.md Appendix B.

  proj/tests/test_solve_stage.cpp   solve / transpose_solve / reduced solves / refine
  proj/tests/test_factor_ds.cpp     factorize: tips, DS identity, reduced levels
  proj/tests/test_acceptance.cpp    the acceptance criteria (ACCEPTANCE ... PASS lines)

Excluded: the acceptance suite's "accuracy study against condition number"
case shells out to the reference CLI (proj/tools/spike_cli.cpp, out of scope
per SURVEY.md section 2; not built), so it cannot run.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXCLUDE = {"test_acceptance": ["accuracy study against condition number"]}


@pytest.mark.parametrize("suite", ["test_solve_stage", "test_factor_ds", "test_acceptance"])
def test_reference_suite_passes(spk, suite, tmp_path):
    exe = os.path.join(ROOT, "oracle", "_ref", "suite_" + suite)
    if not os.path.exists(exe):
        pytest.skip("reference suites not built (oracle/Makefile suites needs /root/reference)")
    args = [exe]
    if suite in EXCLUDE:
        args.append("--test-case-exclude=" + ",".join(EXCLUDE[suite]))
    r = subprocess.run(args, capture_output=True, text=True, timeout=900, cwd=str(tmp_path))
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "| 0 failed" in r.stdout
    if suite == "test_acceptance":
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("ACCEPTANCE")]
        assert len(lines) == 7 and all(ln.rstrip().endswith("PASS") for ln in lines), lines
