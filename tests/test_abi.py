"""CPU-side checks of the C ABI boundary (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "mpeig_b200.h")).read()
    return sorted(set(re.findall(r"\b(mpeig_[a-z0-9_]+)\s*\(", txt)) - {"mpeig_history_sink"})


def test_library_exports_every_declared_symbol():
    import paper_2302_12528_b200 as mp
    lib = mp.load()
    declared = header_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(mp.SYMBOLS) == declared


def test_header_compiles_as_c():
    """the boundary is plain C: no C++ or torch types."""
    import subprocess
    import tempfile
    src = '#include "mpeig_b200.h"\nint main(void){return (int)sizeof(mpeig_cfg) > 0 ? 0 : 1;}\n'
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.c")
        open(p, "w").write(src)
        r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                            p, "-o", os.path.join(d, "t")], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def test_struct_layouts_match_header():
    """ctypes mirrors agree with the C compiler's layout of the ABI structs."""
    import subprocess
    import tempfile
    from paper_2302_12528_b200 import _lib as L
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "mpeig_b200.h"
int main(void){
 printf("%zu %zu %zu %zu %zu %zu\n", sizeof(mpeig_cfg), sizeof(mpeig_stage_opts),
        sizeof(mpeig_iter_record), sizeof(mpeig_timings), sizeof(mpeig_stage_out), sizeof(mpeig_result));
 return 0;}
'''
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.c")
        open(p, "w").write(src)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), p, "-o", exe], check=True)
        sizes = [int(x) for x in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    ours = [C.sizeof(t) for t in (L.Cfg, L.StageOpts, L.IterRecord, L.Timings, L.StageOut, L.Result)]
    assert sizes == ours


def test_gaussian_stream_bitwise_vs_reference():
    """X0 / sketch stream (rng.cpp:24-56, dense_matrix.hpp:144-161) is bit-exact."""
    import paper_2302_12528_b200 as mp
    from oracle import Oracle, available
    orc = Oracle("ref" if available("ref") else "port")
    for rows, cols, seed in ((1001, 7, 42), (33, 5, 0), (10, 3, 0 ^ 0x9E3779B97F4A7C15)):
        assert np.array_equal(mp.gaussian_matrix(rows, cols, seed), orc.gaussian(rows, cols, seed))


def test_gaussian_parallel_jump_ahead():
    """the multi-threaded jump-ahead fill equals the sequential stream."""
    import paper_2302_12528_b200 as mp
    from oracle import Oracle, available
    orc = Oracle("ref" if available("ref") else "port")
    rows, cols = (1 << 20) + 3, 2  # large enough to take the threaded path, odd length
    a = mp.gaussian_matrix(rows, cols, 2026)
    b = orc.gaussian(rows, cols, 2026)
    assert np.array_equal(a, b)


def test_gaussian_golden_fixture():
    import paper_2302_12528_b200 as mp
    path = os.path.join(ROOT, "tests", "golden", "pcg64.npz")
    if not os.path.exists(path):
        pytest.skip("fixture missing")
    g = np.load(path)
    assert np.array_equal(mp.gaussian_matrix(33, 5, 0), g["gauss_0_33x5"])
    assert np.array_equal(mp.gaussian_matrix(40, 8, 0 ^ 0x9E3779B97F4A7C15), g["gauss_sketch"])


def test_product_fails_loudly_without_gpu():
    """no silent CPU fallback: creating a context without a device raises."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2302_12528_b200 as mp
    with pytest.raises(RuntimeError):
        mp.Context(0)
