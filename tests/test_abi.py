"""The C-ABI library loads and exports exactly what include/*.h declares
(no compute without a GPU)."""
import ctypes as C
import glob
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2510_23264_b200 import engine as eng
from helpers import TINY, TOY

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(cqg_\w+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    lib_path = eng.LIB_PATH
    assert os.path.exists(lib_path), "build libcqg.so first"
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True,
                         text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    missing = declared_functions() - exported
    assert not missing, missing
    eng.load_library()


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", eng.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_graph_matches_reference_numbering(ref):
    for cfg in (TINY, TOY):
        n, src, dst = eng.graph_edges(cfg)
        _, _, _, rs, rd = ref.graph(cfg.fields8())
        assert np.array_equal(src, rs) and np.array_equal(dst, rd)


def test_qkv_split_graph_matches_oracle():
    """libcqg's Q/K/V-split graph (extension) equals the oracle's: sources,
    destinations, receiver components, edge count."""
    from oracle.oracle import Port
    from helpers import SMALL, make
    for cfg in (TINY, TOY, SMALL):
        n, src, dst = eng.graph_edges(cfg, qkv_split=True)
        comp = eng.graph_edge_comp(cfg, qkv_split=True)
        p = Port(cfg, make(cfg)[0].mats, qkv_split=True)
        _, _, _, ps, pd = p.graph()
        assert np.array_equal(src, ps) and np.array_equal(dst, pd)
        assert np.array_equal(comp, p.edge_comp())
        assert np.array_equal(eng.graph_edge_comp(cfg), np.zeros(len(eng.graph_edges(cfg)[1]), np.int32))


def test_sweep_order_matches_reference(ref):
    mask = np.random.RandomState(3).rand(33) < 0.5
    got = eng.sweep_order(TOY, mask)
    want = ref.sweep_order(TOY.fields8(), mask.astype(np.uint8))
    assert np.array_equal(got, want)


def test_bad_config_is_invalid_argument():
    lib = eng.load_library()
    c = eng.CqgConfig(1, 3, 8, 2, 16, 4, 0)  # 3*2 != 8
    nn, ne = C.c_int(), C.c_int()
    rc = lib.cqg_graph_info(C.byref(c), C.byref(nn), C.byref(ne))
    assert rc == 1 and b"n_heads * d_k" in lib.cqg_last_error()


def test_fnv_matches_python():
    from paper_2510_23264_b200 import formats
    data = os.urandom(1000)
    assert eng.fnv1a64(data) == formats.fnv1a64(data)


def test_engine_without_gpu_fails_loudly():
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    from paper_2510_23264_b200 import synth
    with pytest.raises(Exception):
        eng.Engine(synth.random_weights(TINY, 1))
