"""The reference's own test suites (proj/tests/{fir,dft,pipeline,coeff,bench,
acceptance}_test.cpp), compiled unchanged by tests/refsuite/build.py:

  *_cpu  against the reference headers (proves the gtest shim is faithful);
  *_gpu  against the B200 drop-in (include/ppf_dropin: namespace ppf over
         libppfg.so) — the reference's tests exercising the CUDA path.

Binaries are built in the container that has /root/reference and travel to
the GPU box; where they are missing the tests skip. The one exclusion is
Criterion7's ">= 2x speed-up of 4 CPU worker threads over the scalar loop"
(acceptance_test.cpp:286-345): it measures CPU threading, which the drop-in
replaces by CUDA threads, so ppf_fir_reference and ppf_fir_optimized run the
same kernel; its FLOP-accounting half is covered by bench_test.
"""
import os
import re
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "refsuite", "_build")
SUITES = ["fir_test", "dft_test", "pipeline_test", "coeff_test", "bench_test", "acceptance_test"]
EXCLUDE = {"acceptance_test": ["-Criterion7_ThroughputScalingAndFlopAccounting"]}


def run_suite(path, args):
    if not os.path.exists(path):
        pytest.skip(f"{os.path.basename(path)} not built (needs /root/reference at build time)")
    p = subprocess.run([path, *args], capture_output=True, text=True, timeout=900,
                       cwd=os.path.dirname(path))
    m = re.search(r"(\d+) passed, (\d+) failed, (\d+) skipped", p.stdout)
    assert m, p.stdout[-2000:] + p.stderr[-2000:]
    passed, failed, skipped = map(int, m.groups())
    assert failed == 0 and p.returncode == 0, "\n".join(
        l for l in p.stdout.splitlines() if "FAILED" in l or "Failure" in l or "actual" in l)[-4000:]
    assert passed > 0
    return passed, skipped


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_reference_headers(suite):
    run_suite(os.path.join(BUILD, suite + "_cpu"), EXCLUDE.get(suite, []))


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_b200_dropin(suite):
    passed, skipped = run_suite(os.path.join(BUILD, suite + "_gpu"), EXCLUDE.get(suite, []))
    assert skipped == 0
