"""The C-ABI library loads on a CPU-only box and exports every symbol that
include/lmscale.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lmscale.h")


def declared_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"LMSCALE_API\s+[\w\s\*]+?\b(lmscale_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    path = __graft_entry__._load_builder().build()
    return ctypes.CDLL(path), path


def test_header_declares_the_boundary():
    fns = declared_functions()
    for name in ["lmscale_init", "lmscale_unique", "lmscale_sync_embedding_grad",
                 "lmscale_apply_sparse_update"]:
        assert name in fns      # BASELINE.json north_star names these four
    assert len(fns) >= 15


def test_library_exports_every_declared_symbol(lib):
    handle, path = lib
    for name in declared_functions():
        assert hasattr(handle, name), name
    out = subprocess.check_output(["nm", "-D", "--defined-only", path], text=True)
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert exported == set(declared_functions()), exported ^ set(declared_functions())


def test_binding_names_match_header(lib):
    from paper_1810_10045_b200 import lmscale
    assert sorted(lmscale.EXPORTED) == declared_functions()
    assert lmscale.version().startswith("lmscale")
    assert lmscale._status_string(2).decode() == "token id >= vocab"
    assert lmscale._status_string(lmscale.CONSISTENCY).decode() == "U_g or I^ differs across ranks"


def test_init_rejects_bad_config_without_touching_gpu(lib):
    from paper_1810_10045_b200 import lmscale
    h = ctypes.c_void_p()
    bad = lmscale.Config(0, 10, 4, 1, 0, 0, 0)   # vocab = 0
    assert lmscale._init(ctypes.byref(bad), None, ctypes.byref(h)) == lmscale.INVALID_ARG
    bad = lmscale.Config(10, 10, 4, 2, 2, 0, 0)  # rank >= world
    assert lmscale._init(ctypes.byref(bad), None, ctypes.byref(h)) == lmscale.INVALID_ARG
    assert not h.value


def test_sm100a_code_in_library(lib):
    _, path = lib
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("policy", ["distinct", "same", "log2", "loge", "log10", "power"])
def test_plan_seeds_host_logic_matches_oracle(lib, policy):
    """lmscale_plan_seeds is host-only (no GPU): same groups and seeds as the
    oracle's plan for every G up to 130 (Sec. 3.2, R16)."""
    import oracle
    from paper_1810_10045_b200 import lmscale
    for G in list(range(1, 70)) + [100, 128, 130]:
        got = lmscale.plan_seeds(G, policy, 0.64, master_seed=181010045)
        want = oracle.plan_seeds(G, policy, alpha=0.64, master_seed=181010045)
        assert got == (want[0], want[1]), (G, policy)
    with pytest.raises(lmscale.LmscaleError):
        lmscale.plan_seeds(8, "power", 1.5)


def test_product_path_never_touches_the_oracle():
    """The product package (paper_1810_10045_b200/: binding + CUDA sources)
    neither imports nor links the CPU oracle, and the binding has no CPU
    fallback: it loads liblmscale.so or raises."""
    import pathlib
    import re
    pkg = pathlib.Path(__file__).resolve().parent.parent / "paper_1810_10045_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = f.read_text()
        assert not re.search(r"^\s*(import|from)\s+oracle", text, re.M), f
        assert "liboracle" not in text and "oracle_" not in text, f
    binding = (pkg / "lmscale.py").read_text()
    assert "CDLL" in binding
