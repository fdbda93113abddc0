"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol include/hv.h declares,
the ctypes structs match the header's field order, and creating a context without a device fails loudly
(HV_ECUDA) instead of falling back to the CPU."""
import ctypes
import os
import re

import pytest

import paper_2507_10804_b200 as hv
from paper_2507_10804_b200 import build as hvbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hv.h")


def declared_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"HV_API\s+[\w\s\*]+?\b(hv_\w+)\s*\(", txt)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for name in ("hv_create", "hv_destroy", "hv_forward", "hv_gradient", "hv_hessvec", "hv_psido_apply",
                 "hv_gradient_hessvec", "hv_set_stream", "hv_get_stats", "hv_last_error"):
        assert name in fns


def test_library_builds_and_exports_every_declared_symbol():
    hvbuild.build()
    L = hv.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
        assert ctypes.cast(getattr(L, name), ctypes.c_void_p).value


def test_config_struct_matches_header_order():
    txt = open(HEADER).read()
    body = txt[txt.index("typedef struct {"):txt.index("} hv_config;")]
    names = re.findall(r"\b(\w+)\s*[,;]", re.sub(r"/\*.*?\*/", "", body, flags=re.S))
    names = [n for n in names if n not in ("int32_t", "float", "size_t")]
    assert names == [f for f, _ in hv.HvConfig._fields_]
    sbody = txt[txt.index("int64_t kernel_launches"):txt.index("} hv_stats;")]
    snames = re.findall(r"\b(\w+)\s*;", re.sub(r"/\*.*?\*/", "", sbody, flags=re.S))
    assert snames == [f for f, _ in hv.HvStats._fields_]


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import workloads
    with pytest.raises(hv.HVError) as e:
        hv.Solver.from_workload(workloads.config(0))
    assert e.value.status == hv.HV_ECUDA


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2507_10804_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), f
                assert "oracle/" not in src.replace("`oracle/`", ""), f


def test_nccl_helpers_without_gpu():
    """The in-library NCCL path dlopens libnccl.so.2: a unique id is available on the CPU host; creating a
    communicator without a device fails loudly (HV_ECUDA) instead of hanging or falling back."""
    import torch
    uid = hv.nccl_unique_id()
    assert len(uid) == 128 and any(uid)
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(hv.HVError) as e:
        hv.nccl_comm_create(1, 0, uid, 0)
    assert e.value.status == hv.HV_ECUDA
    with pytest.raises(ValueError):
        hv.nccl_comm_create(1, 0, b"short", 0)
