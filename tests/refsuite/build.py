#!/usr/bin/env python
"""Compile the reference's OWN test suites, unchanged, from
/root/reference/proj/tests (nothing is copied into this repo):

  <suite>_gpu : against the B200 drop-in (include/ppf_dropin -> namespace ppf
                over libppfg.so). Runs on the GPU box (tests/test_refsuite.py).
  <suite>_cpu : against the reference headers themselves — proves the gtest
                shim runs the suites faithfully (they pass here, on CPU).

Binaries go to tests/refsuite/_build/ (git-ignored, travels to the GPU box
with the snapshot). Only possible where /root/reference exists.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_TESTS = "/root/reference/proj/tests"
REF_INC = "/root/reference/proj/include"
OUT = os.path.join(HERE, "_build")
SUITES = ["fir_test", "dft_test", "pipeline_test", "coeff_test", "bench_test", "acceptance_test"]


def json_dir():
    import site
    for p in site.getsitepackages():
        d = os.path.join(p, "include", "cudnn_frontend", "thirdparty", "nlohmann")
        if os.path.isdir(d):
            return d
    raise SystemExit("nlohmann/json.hpp not found")


def build(which=("gpu", "cpu"), suites=SUITES):
    if not os.path.isdir(REF_TESTS):
        print("no /root/reference: nothing to build", file=sys.stderr)
        return False
    os.makedirs(OUT, exist_ok=True)
    common = ["g++", "-std=gnu++20", "-O2", "-pthread", "-include", "algorithm",
              "-I", os.path.join(HERE), "-I", json_dir(), "-w"]
    lib_dir = os.path.join(ROOT, "paper_1411_3656_b200")
    deps = [os.path.join(HERE, "gtest", "gtest.h")] + [
        os.path.join(dp, f) for d in ("include/ppf_gpu", "include/ppf_dropin/ppf", "include")
        for dp in [os.path.join(ROOT, d)] for f in os.listdir(dp) if f.endswith((".h", ".hpp"))]

    def fresh(out, src):
        if not os.path.exists(out):
            return False
        t = os.path.getmtime(out)
        return all(os.path.getmtime(p) <= t for p in deps + [src, os.path.join(REF_TESTS,
                                                                               "testing_util.hpp")])

    for s in suites:
        src = os.path.join(REF_TESTS, s + ".cpp")
        if "gpu" in which and not fresh(os.path.join(OUT, s + "_gpu"), src):
            cmd = common + ["-I", os.path.join(ROOT, "include", "ppf_dropin"), "-I",
                            os.path.join(ROOT, "include"), src, "-o", os.path.join(OUT, s + "_gpu"),
                            "-L", lib_dir, "-lppfg",
                            "-Wl,-rpath,$ORIGIN/../../../paper_1411_3656_b200"]
            subprocess.check_call(cmd)
        if "cpu" in which and not fresh(os.path.join(OUT, s + "_cpu"), src):
            cmd = common + ["-march=native", "-I", REF_INC, src, "-o", os.path.join(OUT, s + "_cpu")]
            subprocess.check_call(cmd)
    return True


if __name__ == "__main__":
    build(which=tuple(sys.argv[1:]) or ("gpu", "cpu"))
    print(OUT)
