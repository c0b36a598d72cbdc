"""cs_introsort.h (the device fit's sort) == the host's std::sort, permutation
for permutation, on tie-heavy, sorted, reversed, organ-pipe and
median-of-three-adversarial inputs (the last reach the heap-sort fallback).
The GBDT fit's prefix sums run in this order (gbdt.cpp:60-76)."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_introsort_matches_std_sort(tmp_path):
    exe = tmp_path / "introsort_check"
    subprocess.run(["g++", "-O2", "-std=c++17", os.path.join(HERE, "native", "introsort_check.cpp"),
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    assert out.startswith("ok "), out
