"""CPU tier: the C-ABI library builds, loads and exports every declared entry
point; the FP64 kernels contain no contracted multiply-adds; the product has
no CPU fallback and never touches the oracle."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, cuda_visible
from paper_2510_01592_b200 import native

HEADERS = ["voxplane_b200.h", "voxplane_scene.h"]


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vp_[a-z0-9_]+)\s*\(", src)))


def exported():
    out = subprocess.run(["nm", "-D", "--defined-only", native.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


@pytest.mark.parametrize("header", HEADERS)
def test_every_declared_symbol_is_exported(header):
    names = declared(header)
    assert len(names) > 5
    missing = [n for n in names if n not in exported()]
    assert missing == []
    L = native.lib()
    for n in names:
        getattr(L, n)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


@pytest.mark.parametrize("src", ["k_map.cu", "k_segment.cu"])
def test_no_fp64_contraction_in_kernels(src, tmp_path):
    # bit-exactness needs every a*b+c rounded twice, like the reference built
    # with -ffp-contract=off; IEEE div/sqrt expansions are allowed (they are
    # correctly rounded), user-level fma.rn.f64 is not.
    ptx = tmp_path / (src + ".ptx")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=compute_100a", "-O3", "-std=c++17",
                    "-fmad=false", "-I", os.path.join(ROOT, "include"), "-ptx",
                    os.path.join(ROOT, "paper_2510_01592_b200", "csrc", src), "-o", str(ptx)], check=True)
    text = ptx.read_text()
    assert "fma.rn.f64" not in text
    assert "div.rn.f64" in text


def test_build_flags_keep_fmad_off():
    import __graft_entry__ as g
    assert "-fmad=false" in g.NVCC_FLAGS and "arch=compute_100a,code=sm_100a" in g.NVCC_FLAGS


@pytest.mark.skipif(cuda_visible(), reason="checks the no-device error path")
def test_no_device_fails_loudly():
    with pytest.raises(native.VpError) as e:
        native.Grid(0.01, (8, 8, 8), (0, 0, 0))
    assert e.value.code == native.VP_ENODEV


def test_invalid_grid_arguments_raise_before_device():
    # VoxelGrid constructor contract (voxel_grid.cpp:21-22) holds on any box
    for res, ext in [(0.0, (4, 4, 4)), (0.01, (4, 0, 4)), (-1.0, (4, 4, 4))]:
        with pytest.raises(native.InvalidArgument):
            native.Grid(res, ext, (0, 0, 0))


def test_product_never_imports_or_links_the_oracle():
    pkg = os.path.join(ROOT, "paper_2510_01592_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "liboracle" not in text and "cpu_oracles" not in text and "voxplane_oracle" not in text
    ldd = subprocess.run(["ldd", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in ldd and "voxplane_ref" not in ldd


def test_default_params_match_reference_defaults():
    p = C.cast(C.create_string_buffer(C.sizeof(native.PipelineParams)), C.POINTER(native.PipelineParams)).contents
    native.lib().vp_default_params(C.byref(p))
    q = native.default_params()
    assert bytes(p) == bytes(q)
    assert (p.seg.neighbor_radius, p.seg.min_neighbors, p.seg.min_cluster_size) == (1, 3, 30)
    assert (p.seg.max_angle_deg, p.seg.distance_th, p.ransac.iterations, p.ransac.inlier_eps) == (15.0, 0.05, 100, 0.01)
    assert np.isclose(p.min_polygon_area, 0.002) and p.refine == 1
