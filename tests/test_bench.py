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
