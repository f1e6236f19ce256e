"""CPU checks of the boundary: libgs.so builds for sm_100a, loads, and exports every symbol
include/gs.h declares (no compute calls — there is no GPU here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_04335_b200 import build
    path = build.build()
    import paper_2604_04335_b200 as gs
    return gs.load(path)


def test_header_declares_the_boundary():
    names = _declared()
    for required in ("gs_init", "gs_model_create", "gs_submit", "gs_run_steps", "gs_preempt",
                     "gs_resume", "gs_query", "gs_read_latent", "gs_release", "gs_destroy"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_binding_covers_header():
    import paper_2604_04335_b200 as gs
    assert sorted(gs._SIG) == _declared()


def test_sm100a_cubin_with_tcgen05_and_tma(lib):
    so = os.path.join(ROOT, "paper_2604_04335_b200", "libgs.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out or "UTCQMMA" in out      # tcgen05.mma
    assert "UTMALDG" in out                           # TMA loads
    assert "LDTM" in out and "STTM" in out            # tcgen05.ld / tcgen05.st
    assert "HMMA" not in out.replace("UTCHMMA", "")   # no legacy mma.sync path


def test_no_oracle_on_product_path():
    pkg = os.path.join(ROOT, "paper_2604_04335_b200")
    for dirpath, _d, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
