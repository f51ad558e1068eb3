"""The C++ drop-in (include/sdfrecon_gpu.hpp) used exactly as a reference
maintainer would: oracle/_ref/dropin_test runs the reference's own
sdfrecon::render_image / sdfrecon::train (CPU) and the sdfrecon_gpu
equivalents (GPU) on the same inputs (built where /root/reference exists;
the prebuilt binary travels with the repo)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")

pytestmark = pytest.mark.gpu


def test_cpp_dropin_matches_reference():
    assert os.path.exists(BIN), "oracle/_ref/dropin_test not built (make -C oracle dropin)"
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600, check=True).stdout
    kv = {l.split()[0]: l.split()[1:] for l in out.strip().splitlines()}
    assert float(kv["render_color_maxdiff"][0]) <= 1e-4
    assert float(kv["render_alpha_maxdiff"][0]) <= 1e-5
    assert kv["out_of_range_thrown"] == ["1"]
    assert kv["train_steps"][0] == kv["train_steps"][1] == "40"
    assert abs(float(kv["train_psnr"][0]) - float(kv["train_psnr"][1])) <= 1e-3
    assert kv["train_tiles"][0] == kv["train_tiles"][1]
    assert float(kv["train_raw_maxdiff"][0]) <= 1e-3 * float(kv["train_raw_maxdiff"][2])
    assert kv["train_cursor"][0] == kv["train_cursor"][1]
    assert kv["log_lines"][0] == kv["log_lines"][1] == "40"
    # evaluation drop-ins: chamfer bit-exact, psnr_masked of a render to 1e-3 dB
    assert [l for l in out.splitlines() if l.startswith("chamfer_equal")] == ["chamfer_equal 1"] * 2
    assert abs(float(kv["eval_psnr"][0]) - float(kv["eval_psnr"][1])) <= 1e-3
