"""The drop-in on the reference side: integration/acdc_gpu.cpp
is the translation unit a maintainer adds to circuitquant. It is compiled
against the reference's own headers (proj/include) and linked with the
reference objects compiled in place (oracle/Makefile) plus libcqg.so
(integration/Makefile -> oracle/_ref/integration/check_acdc_gpu).

* CPU: it compiles and links, libcqg's entry points resolve from libcqg.so,
  and the driver's stock leg (the reference's own run_acdc) runs on toy.
* GPU: the reference's loop with the scoring block on libcqg.so (run_acdc_gpu)
  returns the same CircuitResult as the stock run_acdc (acdc.cpp:23-88) on
  BASELINE config 1 (toy, PAHQ 8-bit, tau = 0.01): identical final mask,
  steps, per-iteration edge records and kept flags.
"""
import json
import os
import subprocess

import pytest

from paper_2510_23264_b200 import formats, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "integration", "check_acdc_gpu")
TOY = formats.ModelConfig(2, 4, 128, 32, 512, 16, 1, 0)


def toy_files(tmp_path):
    w = synth.random_weights(TOY, 1)
    ds = synth.random_dataset(TOY, 16, 2)
    wp, dp = str(tmp_path / "weights.bin"), str(tmp_path / "dataset.jsonl")
    formats.save_weights(w, wp)
    formats.save_dataset_jsonl(ds, dp)
    return wp, dp


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj"), reason="needs the reference sources")
def test_shim_compiles_and_links_against_reference(tmp_path):
    subprocess.run(["make", "-C", os.path.join(ROOT, "integration")], check=True, capture_output=True)
    assert os.path.exists(BIN)
    und = subprocess.run(["nm", "-u", BIN], capture_output=True, text=True).stdout
    for sym in ("cqg_create", "cqg_set_dataset", "cqg_score_edges", "cqg_last_error", "cqg_destroy"):
        assert sym in und, sym  # resolved from libcqg.so at load time
    ldd = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libcqg.so" in ldd and "not found" not in ldd.split("libcqg.so")[1].split("\n")[0]
    wp, dp = toy_files(tmp_path)
    r = subprocess.run([BIN, wp, dp, "0.01", "--stock-only"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert json.loads(r.stdout)["stock_steps"] >= 1


@pytest.mark.gpu
def test_reference_loop_with_gpu_scoring_matches_stock(tmp_path):
    if not os.path.exists(BIN):
        pytest.skip("integration binary not built (make -C integration, needs /root/reference)")
    wp, dp = toy_files(tmp_path)
    r = subprocess.run([BIN, wp, dp, "0.01"], capture_output=True, text=True, timeout=900)
    out = json.loads(r.stdout.strip().splitlines()[-1])
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "integration_toy.json"), "w"), indent=1)
    assert r.returncode == 0, r.stdout + r.stderr
    assert out["same_final_mask"] and out["same_steps"] and out["same_records"], out
    assert out["max_rel_score_diff"] <= 1e-9, out
