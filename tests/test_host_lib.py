"""The C-ABI library (paper_2103_10453_b200/libplse_b200.so) on a CPU-only box:
it loads, exports every entry point include/plse_b200.h declares, its host
helpers match the reference (golden vectors), errors map like the reference's
exceptions, and device entry points fail loudly (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = np.load(os.path.join(ROOT, "tests", "golden", "ref_golden.npz"))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "plse_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(plse_[a-z_0-9]+)\s*\(", text)) - {"plse_generation_cb"})


def test_library_exports_every_declared_symbol(plse):
    lib = ctypes.CDLL(plse.lib_path())
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.plse_abi_version() == 2


def test_oracle_library_is_not_linked_into_product(plse):
    """the product .so must not depend on the checker"""
    data = open(plse.lib_path(), "rb").read()
    assert b"liboracle" not in data and b"or_improve" not in data and b"libplse_ref" not in data


@pytest.mark.parametrize("key", [k for k in G.files if k.startswith("inst_")])
def test_generate_and_preprocess_match_reference(plse, key):
    _, n, r, s = key.split("_")
    grid = plse.generate_instance(int(n), float(r), int(s))
    assert np.array_equal(grid, G[key])
    g = plse.preprocess(grid)
    gold = G[key.replace("inst_", "graph_")]
    nv, l = int(gold[0]), int(gold[1])
    assert (g.vertex_count, g.l) == (nv, l)
    assert np.array_equal(g.cell_row, gold[2:2 + nv]) and np.array_equal(g.cell_col, gold[2 + nv:2 + 2 * nv])
    tail = gold[2 + 2 * nv:]
    adj_len = int(tail[nv])  # adj_off[nv]
    dom_off = tail[nv + 1 + adj_len: nv + 1 + adj_len + nv + 1]
    assert np.array_equal(g.dom_offsets, dom_off)
    assert np.array_equal(g.dom, tail[nv + 1 + adj_len + nv + 1:].astype(np.uint16))
    pre = {(int(a), int(b)): int(c) for a, b, c in g.prefilled}
    assert pre == {(i // int(n), i % int(n)): int(v) for i, v in enumerate(grid.reshape(-1)) if v}


def test_parse_serialize_round_trip(plse):
    grid = G["inst_10_0.3_606"]
    assert np.array_equal(plse.parse_instance(plse.serialize_instance(grid)), grid)
    assert np.array_equal(plse.parse_instance("\n\n3\n1 0 0\n\n2 0 0\n0 0 3\n"),
                          np.array([[1, 0, 0], [2, 0, 0], [0, 0, 3]], np.uint16))


@pytest.mark.parametrize("text,msg", [("", "line 1: unexpected end of input"), ("x\n", "line 1: malformed header"),
                                      ("2\n1 2\n", "line 3: unexpected end"), ("2\n1 3\n0 0\n", "symbol out of range"),
                                      ("2\n1 1\n0 0\n", "line 2: duplicate symbol 1 in row 0"),
                                      ("2\n1 0 0\n0 0\n", "trailing tokens")])
def test_parse_errors_carry_line_numbers(plse, text, msg):
    """instance.hpp:107-170 / test_instance.cpp:18-41"""
    with pytest.raises(RuntimeError, match=msg):
        plse.parse_instance(text)


def test_argument_errors_map_to_value_error(plse):
    with pytest.raises(ValueError):
        plse.generate_instance(0, 0.5, 1)
    with pytest.raises(ValueError):
        plse.generate_instance(5, 1.0, 1)
    g = plse.preprocess(G["inst_10_0.3_606"])
    for bad in (dict(p=1), dict(gamma=1.0), dict(beta=5.0), dict(alpha=-1.0)):
        with pytest.raises(ValueError):
            plse.DevicePopulation(g, plse.SolverConfig(**{"p": 8, **bad}))


def test_device_path_fails_loudly_without_gpu(plse):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    g = plse.preprocess(G["inst_10_0.3_606"])
    with pytest.raises(plse.PlseCudaError):
        plse.DevicePopulation(g, plse.SolverConfig(p=8))
    with pytest.raises(plse.PlseCudaError):
        plse.run(G["inst_10_0.3_606"], plse.SolverConfig(p=8, generation_limit=1))


def test_unsupported_requests(plse):
    with pytest.raises(ValueError, match="unknown variant"):
        plse.run(G["inst_10_0.3_606"], plse.SolverConfig(p=8, variant=7))
    with pytest.raises(ValueError, match="phase budgets"):
        plse.run(G["inst_10_0.3_606"], plse.SolverConfig(p=8, variant=plse.MPMA, phase2_iters=-1))
    big = np.zeros((130, 130), np.uint16)
    with pytest.raises(NotImplementedError):
        plse.DevicePopulation(plse.preprocess(big), plse.SolverConfig(p=4))


def test_trivial_instance_runs_without_device(plse):
    """engine.hpp:143-146: |V| = 0 finalises as 'trivial' before any device work"""
    full = np.array([[1, 2], [2, 1]], np.uint16)
    r = plse.run(full, plse.SolverConfig(p=4))
    assert r.stop_reason == "optimal" and r.best_score == 4 and r.vertex_count == 0


def test_lsc_instance_matches_reference_builder(plse):
    """config C5's LSC stand-in (builders.hpp:30-58)"""
    assert np.array_equal(plse.lsc_instance(20, 0.4, 7), G["lsc_20_0.4_7"])
    assert np.array_equal(plse.lsc_instance(70, 0.4, 7), G["lsc_70_0.4_7"])


def test_raw_abi_rejects_null_and_bad_arguments(plse):
    """Every context entry point rejects a NULL context with PLSE_ERR_INVALID (no crash, no device
    work) and leaves a message in plse_last_error(NULL); host helpers reject NULL buffers."""
    lib = ctypes.CDLL(plse.lib_path())
    lib.plse_last_error.restype = ctypes.c_char_p
    INVALID = 1
    nul = ctypes.c_void_p()
    buf = (ctypes.c_uint16 * 16)()
    i32 = ctypes.c_int32()
    i64 = ctypes.c_int64()
    calls = {
        "plse_init_population": (nul,),
        "plse_full_distances": (nul,),
        "plse_improve": (nul, ctypes.c_uint64(1), ctypes.byref(i64), ctypes.byref(i32), ctypes.byref(i32)),
        "plse_distances": (nul,),
        "plse_update": (nul, ctypes.byref(i32), ctypes.byref(i32), nul),
        "plse_reset_exclusion": (nul,),
        "plse_offspring": (nul, ctypes.c_uint64(1)),
        "plse_export_elites": (nul, ctypes.c_int32(1), nul, nul),
        "plse_import_migrants": (nul, ctypes.c_int32(1), nul),
        "plse_get_stats": (nul, ctypes.c_int32(0), nul, nul, nul),
        "plse_get_counters": (nul, nul),
        "plse_timer_start": (nul,),
        "plse_get_colors": (nul, ctypes.c_int32(0), buf),
        "plse_get_row": (nul, ctypes.c_int32(0), ctypes.c_int32(0), buf),
        "plse_to_grid": (nul, buf, buf),
        "plse_solve_exact": (nul, ctypes.c_int64(10), ctypes.byref(i32), ctypes.byref(i32), ctypes.byref(i64), buf),
        "plse_verify_certificate": (ctypes.c_int32(2), nul, ctypes.c_int32(2), nul, ctypes.byref(i32),
                                    ctypes.byref(i32), nul, ctypes.c_int64(0), ctypes.byref(i64)),
        "plse_preprocess": (ctypes.c_int32(2), nul, ctypes.byref(nul)),
        "plse_solve": (ctypes.c_int32(2), nul, nul, nul, nul, nul, nul),
    }
    for name, args in calls.items():
        rc = getattr(lib, name)(*args)
        assert rc == INVALID, (name, rc)
        assert lib.plse_last_error(None), name
