"""CPU-side checks of the C-ABI boundary (-m "not gpu"): the library loads,
exports every symbol include/be.h declares, pure helpers work without a
GPU, and device calls fail loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "be.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(be_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_1912_01703_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_1912_01703_b200 import build
        build.build()
    return _lib.lib()


def test_header_declares_boundary():
    names = declared_functions()
    for must in ["be_init", "be_tensor_create", "be_release", "be_op", "be_backward", "be_sgd_step",
                 "be_alloc_stats", "be_empty_cache", "be_ddp_attach", "be_dist_init"]:
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    from paper_1912_01703_b200 import _lib
    assert sorted(_lib.EXPORTED) == declared_functions()


def test_round_size_pure(lib):
    # PAPER.md:198 / SPEC S:371-373
    import json
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))["round_size"]
    for n, r in g["cases"]:
        assert lib.be_round_size(ctypes.c_uint64(n)) == r


def test_calls_before_init_fail_loudly(lib):
    from paper_1912_01703_b200 import api as T, BeError
    with pytest.raises(BeError) as e:
        T.empty((4,), "f32")
    assert e.value.name in ("BE_E_NOT_INIT", "BE_E_CUDA")


def test_init_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1912_01703_b200 import api as T, BeError
    with pytest.raises(BeError):
        T.init(0)


def test_sass_contains_tcgen05_and_tma():
    """The GEMM is tcgen05 + TMA (UTC*MMA / UTMALDG / LDTM in SASS)."""
    import shutil
    import subprocess
    from paper_1912_01703_b200 import _lib
    if not shutil.which("cuobjdump") and not os.path.exists("/usr/local/cuda/bin/cuobjdump"):
        pytest.skip("no cuobjdump")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert re.search(r"UTC\w*MMA", out) and "UTMALDG" in out and "LDTM" in out
