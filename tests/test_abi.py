"""The C-ABI library: loads without a GPU, exports every symbol declared in
include/macrofacet_b200.h, and the ctypes mirror matches the C layout
(checked by compiling the header with gcc).  CPU only; no compute calls."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2603_00280_b200 import _lib, build

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "macrofacet_b200.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(build.OUT):
        build.build()
    return ctypes.CDLL(build.OUT)


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mf_[a-z_0-9]+)\s*\(", text)))


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert {"mf_query_batch", "mf_render", "mf_trace_paths", "mf_transmittance",
            "mf_last_error"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", build.OUT], capture_output=True,
                         text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n
    assert set(names) == set(_lib.SIGNATURES), "ctypes SIGNATURES out of sync with the header"


def test_abi_version_and_error_string(lib):
    lib.mf_abi_version.restype = ctypes.c_int
    assert lib.mf_abi_version() == _lib.ABI_VERSION == 4
    lib.mf_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.mf_last_error(), bytes)


def test_parameter_errors_without_gpu(lib):
    """Validation happens before any CUDA call: bad media map to
    ParameterDomainError through the status code."""
    lib.mf_render.restype = ctypes.c_int
    scene = _lib.MfScene()
    params = _lib.MfRenderParams()
    params.spp = 0
    params.max_bounces = 1
    params.nranks = 1
    rc = lib.mf_render(ctypes.byref(scene), ctypes.byref(params), ctypes.c_void_p(1), None, None)
    assert rc == 1
    lib.mf_last_error.restype = ctypes.c_char_p
    assert b"spp" in lib.mf_last_error()


STRUCTS = {
    "mf_medium": _lib.MfMedium, "mf_primitive": _lib.MfPrimitive, "mf_camera": _lib.MfCamera,
    "mf_scene": _lib.MfScene, "mf_render_params": _lib.MfRenderParams, "mf_stats": _lib.MfStats,
    "mf_query_in": _lib.MfQueryIn, "mf_query_out": _lib.MfQueryOut,
}


def test_struct_layout_matches_header(tmp_path):
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, ct in STRUCTS.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in ct._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True,
                                                  text=True).stdout.splitlines())
    for cname, ct in STRUCTS.items():
        assert int(got[cname]) == ctypes.sizeof(ct), cname
        for fname, _ in ct._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(ct, fname).offset, (cname, fname)


def test_sm100a_code_in_library():
    out = subprocess.run(["cuobjdump", "--list-elf", build.OUT], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
STRUCTS["mf_grid_field"] = _lib.MfGridField
STRUCTS["mf_gp_grid"] = _lib.MfGpGrid


def test_async_render_parameter_errors_without_gpu(lib):
    """mf_render_async validates before any CUDA call and hands out no
    ticket on an error; mf_render_finish rejects a null ticket."""
    lib.mf_render_async.restype = ctypes.c_int
    lib.mf_render_finish.restype = ctypes.c_int
    scene = _lib.MfScene()
    params = _lib.MfRenderParams()
    params.spp = 1
    params.max_bounces = 0
    params.nranks = 1
    h = ctypes.c_void_p(123)
    rc = lib.mf_render_async(ctypes.byref(scene), ctypes.byref(params), ctypes.c_void_p(1),
                             ctypes.byref(h), None)
    assert rc == 1 and not h.value
    assert lib.mf_render_finish(None, None) == 1
