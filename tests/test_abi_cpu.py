"""No-GPU checks of the boundary: libbagel.so loads, exports every symbol that
include/bagel.h declares, the binding exposes the same names, and the product
package never imports the oracle."""
import ast
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "bagel.h")
PKG = os.path.join(ROOT, "paper_2202_13638_b200")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2202_13638_b200 import build

    return build.build_library()


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("gp_load", "love_cache_build", "rollout_cost_and_grad", "policy_configure", "reward_configure",
              "bagel_create", "bagel_destroy", "bagel_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_library_loads_and_binding_names_match(libpath):
    from paper_2202_13638_b200 import bagel

    L = bagel.lib()
    for n in declared_functions():
        assert hasattr(L, n), n
    assert sorted(bagel.EXPORTS) == sorted(declared_functions())


def test_library_is_sm100a_and_uses_no_cuda_fallback(libpath):
    out = subprocess.check_output(["cuobjdump", "--list-elf", libpath], text=True)
    assert "sm_100a" in out


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if not f.endswith(".py"):
                continue
            tree = ast.parse(open(os.path.join(dirpath, f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert all(not a.name.startswith("oracle") for a in node.names), f
                if isinstance(node, ast.ImportFrom):
                    assert not (node.module or "").startswith("oracle"), f
    for dirpath, _, files in os.walk(os.path.join(PKG, "csrc")):
        for f in files:
            src = open(os.path.join(dirpath, f)).read()
            assert "bagel_oracle" not in src and "orc_" not in src, f


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2202_13638_b200 import bagel

    monkeypatch.setattr(bagel, "_lib", None)
    monkeypatch.setattr(bagel, "LIB", str(tmp_path / "nope.so"))
    with pytest.raises(RuntimeError, match="missing"):
        bagel.lib()


def test_stale_library_is_detected_by_content(monkeypatch):
    """Staleness is the sources' content hash (compiled into the library and stored next to it), not
    file mtimes: a library built from other sources is never reused."""
    from paper_2202_13638_b200 import bagel, build

    assert build.up_to_date()
    assert bagel.lib().bagel_build_hash().decode() == build.source_hash()
    monkeypatch.setattr(build, "built_hash", lambda: "0" * 64)
    assert not build.up_to_date()


def test_every_declaration_states_its_errors_and_core_calls_cite_the_paper():
    """include/bagel.h contract: each entry point documents its error behaviour; the calls of the
    path and around it cite the passage that defines the operation."""
    src = open(HEADER).read()
    blocks = re.finditer(r"/\*(.*?)\*/\s*((?:#define[^\n]*\n\s*)*(?:(?:const\s+)?\w+\s*\*?\s*\w+\s*\([^;]*\);\s*)+)",
                         src, flags=re.S)
    seen = set()
    for m in blocks:
        comment = m.group(1)
        names = re.findall(r"(\w+)\s*\(", re.sub(r"#define[^\n]*\n", "", m.group(2)))
        seen.update(names)
        assert re.search(r"Errors?:|E_ARG|E_CUDA|E_STATE", comment), names
        core = {"gp_load", "love_cache_build", "exact_cache_build", "gp_target_mode", "policy_configure",
                "reward_configure", "rollout_cost_and_grad", "bagel_sample_states", "policy_adam_step",
                "gp_log_marginal_likelihood", "bagel_gp_predict", "bagel_rollout_trace"}
        if core & set(names):
            assert re.search(r"P:\d+", comment), names
    assert set(declared_functions()) <= seen
