"""The C++ drop-in (paper_2601_09258_b200/dropin) against the reference's own
headers and its own benchmark harness (simkit::evaluate_trial, BASELINE
config 4: per-strategy confusion counts, F1, FPR, lag, RCA top class)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
DEMO_REF = os.path.join(ROOT, "oracle", "_ref", "dropin_demo_ref")
DEMO_GPU = os.path.join(ROOT, "oracle", "_ref", "dropin_demo_gpu")
NLOHMANN = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_dropin_compiles_against_reference_headers():
    r = subprocess.run(["g++", "-std=gnu++20", "-fsyntax-only", f"-I{REF_INC}",
                        f"-I{ROOT}/oracle/shim", f"-I{NLOHMANN}", f"-I{ROOT}/include",
                        f"{ROOT}/paper_2601_09258_b200/dropin/cyclescope_dropin.cpp"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]


def test_dropin_refuses_without_device():
    import torch
    if torch.cuda.is_available() or not os.path.exists(DEMO_GPU):
        pytest.skip("needs the prebuilt demo and no GPU")
    r = subprocess.run([DEMO_GPU, "1"], capture_output=True, text=True)
    assert r.returncode != 0 and "no CPU fallback" in r.stderr


@pytest.mark.gpu
def test_evaluate_trial_identical_with_gpu_dropin():
    """The reference's suite harness with its segmentation / records served by
    the GPU equals the pure reference on 8 trials (one per fault family)."""
    if not (os.path.exists(DEMO_REF) and os.path.exists(DEMO_GPU)):
        pytest.skip("integration demos not built (need /root/reference at build time)")
    ref = subprocess.run([DEMO_REF, "8"], capture_output=True, text=True, timeout=600)
    gpu = subprocess.run([DEMO_GPU, "8"], capture_output=True, text=True, timeout=600)
    assert ref.returncode == 0, ref.stderr[-1000:]
    assert gpu.returncode == 0, gpu.stderr[-1000:]
    assert len(ref.stdout.splitlines()) == 8
    assert gpu.stdout == ref.stdout
