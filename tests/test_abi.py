"""CPU-side checks of the C-ABI boundary (no GPU needed): the library
loads, exports every symbol include/sparseforge_b200.h declares, and its
host-side planner / storage inference / format resolution agree with the
reference's (plan_conversion, infer_storage, resolve_format)."""
import os
import re
import subprocess

import pytest

import paper_2403_05802_b200 as sfg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sparseforge_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sfgx?_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    sfg.load()
    out = subprocess.run(["nm", "-D", "--defined-only", sfg.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT\s+(\S+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert len(declared_symbols()) >= 25


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", sfg.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


FORMATS = ["COO", "CSR", "CSC", "DCSR", "ELL", "BCSR(2,2)", "BCSR(4,4)", "BCSR(16,16)", "BCSR(3,2)", "DOK", "LIL", "BELL(2)", "BELL(4)", "BELL(16)",
           "DIA", "CSB(2)", "CSB(2,3)", "CSB(16)", "CSB(3,2)", "BDIA(2)", "BDIA(3)",
           "C2SR(2)", "C2SR(3)", "DCSC", "DIA-variant", "CISR(2)", "CISR(3)", "CISR-plus(2)", "CISR-plus(5)"]


@pytest.mark.parametrize("fmt", FORMATS)
def test_plan_matches_reference_planner(ref, fmt):
    assert sfg.plan_lines("COO", fmt) == ref.plan("COO", fmt)


@pytest.mark.parametrize("fmt", FORMATS)
def test_storage_explain_matches_reference(ref, fmt):
    assert sfg.storage_explain(fmt) == ref.explain(fmt)


def test_format_resolution():
    f = sfg.resolve_format("BCSR(4)")
    assert (f.kind, f.block_r, f.block_c) == (sfg.KINDS["BCSR"], 4, 4)
    f = sfg.resolve_format("BCSR")
    assert (f.block_r, f.block_c) == (2, 2)  # formats.hpp:49-53 defaults
    f = sfg.resolve_format(" HYB( 8 ) ")
    assert (f.kind, f.threshold) == (sfg.KINDS["HYB"], 8)
    for bad in ["", "FOO", "BCSR(a)", "BCSR(2,2,2)", "CSR("]:
        with pytest.raises(sfg.SfgError) as ei:
            sfg.resolve_format(bad)
        assert ei.value.kind == "Parse", bad


SOURCES = ["CSR", "DCSR", "CSC", "BCSR(2,2)", "BCSR(4,4)", "BCSR(3,2)", "DIA", "CSB(2)", "CSB(2,3)", "CSB(3,2)", "BDIA(2)", "BDIA(3)",
           "DCSC", "DIA-variant"]


@pytest.mark.parametrize("src", SOURCES)
def test_plan_from_compressed_sources_matches_reference(ref, src):
    """planner.hpp:95-252 from a non-COO source: expand the source's levels,
    sort where the target does not, then the target's ops."""
    for dst in FORMATS:
        assert sfg.plan_lines(src, dst) == ref.plan(src, dst), (src, dst)


@pytest.mark.parametrize("src,why", [("ELL", "indirect levels"), ("BELL(2)", "indirect levels"),
                                     ("DOK", "value layout"), ("LIL", "value layout"),
                                     ("C2SR(2)", "value layout"), ("CISR(2)", "indirect levels"),
                                     ("CISR-plus(3)", "indirect levels")])
def test_plan_rejects_sources_like_the_reference(ref, src, why):
    with pytest.raises(sfg.SfgError) as ei:
        sfg.plan_lines(src, "CSR")
    assert ei.value.kind == "UnsupportedSource" and why in str(ei.value)
    with pytest.raises(Exception) as er:
        ref.plan(src, "CSR")
    assert why in str(er.value)


def test_context_without_gpu_fails_loudly():
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(sfg.SfgError) as ei:
        sfg.Context(0)
    assert ei.value.kind == "Cuda"


def test_missing_extension_fails_loudly(monkeypatch):
    # no CPU fallback: without libsfg.so every entry point refuses to run
    monkeypatch.setattr(sfg, "_lib", None)
    monkeypatch.setattr(sfg, "LIB_PATH", sfg.LIB_PATH + ".absent")
    with pytest.raises(ImportError):
        sfg.load()
    with pytest.raises(ImportError):
        sfg.resolve_format("CSR")
