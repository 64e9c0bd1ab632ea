"""CPU-only checks of the C ABI library: it builds for sm_100a, loads, exports
every symbol include/ibnb.h declares, its device constants are the tight
enclosures of the true values, and the product package never touches the
oracle."""
from __future__ import annotations

import ctypes
import math
import os
import re
import subprocess
from fractions import Fraction

import pytest

from tests import hp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ibnb.h")
PKG = os.path.join(ROOT, "paper_2507_01770_b200")


@pytest.fixture(scope="module")
def libpath():
    from paper_2507_01770_b200 import build

    return build.build()


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ib_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("ib_solve", "ib_solve_dev", "ib_eval_boxes", "ib_eval_grad", "ib_branch", "ib_compact_le",
                 "ib_select", "ib_search", "ib_version", "ib_last_error", "ib_solve_workspace_size"):
        assert must in names


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\s[TW]\s+(\S+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    L = ctypes.CDLL(libpath)
    for f in declared_functions():
        getattr(L, f)


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_without_gpu(libpath):
    import paper_2507_01770_b200 as pb

    assert "ibnb" in pb.ib_version()
    assert pb.ib_num_functions() == 11
    # workspace sizing is host-only
    assert pb.solve_workspace_bytes(1, 10) > 0


def test_device_constants_are_tight():
    src = open(os.path.join(PKG, "csrc", "ival.cuh")).read()
    truth = {
        "PI": Fraction(hp.PI),
        "INV_PI": 1 / Fraction(hp.PI),
        "E": Fraction(hp.E),
        "C0_02": Fraction(2, 100),
        "C0_1": Fraction(1, 10),
        "C0_9": Fraction(9, 10),
    }
    for name, v in truth.items():
        lo = float.fromhex(re.search(rf"{name}_LO = ([0-9a-fx.p+-]+)", src).group(1))
        hi = float.fromhex(re.search(rf"{name}_HI = ([0-9a-fx.p+-]+)", src).group(1))
        assert Fraction(lo) <= v <= Fraction(hi), name
        assert math.nextafter(lo, math.inf) == hi, name


def test_product_path_never_uses_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                bad = re.findall(r"(^\s*(import|from)\s+oracle\b|#include\s*[\"<][^\">]*oracle|liboracle|or_(solve|branch|eval))",
                                 txt, flags=re.M)
                assert not bad, (os.path.join(dirpath, f), bad)
