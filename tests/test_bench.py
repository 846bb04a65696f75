"""bench.py's CPU legs (no GPU needed): the reference arm prints one JSON line
with the contract's keys; the GPU arm's argument handling is importable."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "libcqref.so")


@pytest.mark.skipif(not os.path.exists(REF), reason="reference library not built (make -C oracle ref)")
def test_reference_arm_prints_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "toy", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_module_imports():
    sys.path.insert(0, ROOT)
    import bench  # noqa: F401
    assert "gpt2s" in bench.CONFIGS and "toy" in bench.CONFIGS


@pytest.mark.skipif(not os.path.exists(REF), reason="reference library not built (make -C oracle ref)")
def test_reference_arm_is_independent_of_libcqg():
    """The reference arm enumerates edges with the reference's own graph and
    never maps the product library."""
    code = ("import sys; sys.argv=['bench.py']; import bench; "
            "bench.main(['--impl','reference','--config','toy','--steps','1','--warmup','0']); "
            "print('MAPS', 'libcqg' in open('/proc/self/maps').read())")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "MAPS False" in r.stdout, r.stdout[-500:]


@pytest.mark.skipif(not os.path.exists(REF), reason="reference library not built (make -C oracle ref)")
def test_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` without torchrun starts 2 ranks (torch.distributed.run
    on 127.0.0.1); rank 0 prints the one line, and it reports n_gpus 2."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--config", "toy", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    assert json.loads(lines[0])["n_gpus"] == 2


def test_config_block_reports_samples_and_extensions():
    """The workload block names what was measured: strided edge samples
    (configs 4-5 on one GPU), one GPU's item shard, the Q/K/V-split graph and
    the INT8 extension, so a sampled or extension line cannot pass for the
    headline workload."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    a = argparse.Namespace(config="pythia", gpus=1, items=64, qkv_split=True, low="int8")
    c = bench.config_block(a, 80965, 1500)
    assert c["edges_sampled"] == {"scored": 1500, "of": 80965}
    assert c["items"] == 64 and "items_note" in c
    assert "Q/K/V-split" in c["edges"] and c["low_precision"].startswith("int8")
    a = argparse.Namespace(config="gpt2s", gpus=1, items=0, qkv_split=False, low="e4m3")
    c = bench.config_block(a, 11611, 11611)
    assert "edges_sampled" not in c and c["items"] == 64 and "every edge" in c["workload"]
    assert bench.CONFIGS["pythia"]["cfg"].d_k == 128 and bench.CONFIGS["pythia"]["cfg"].seq_len == 32
