"""CPU tests of the C-ABI boundary: the CUDA library builds for sm_100a, loads without a
GPU, exports every entry point include/pathrec_gpu.h declares, and the ctypes mirror's
struct layouts match a C compile of the header.  No compute calls (no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2110_00085_b200 import abi

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "pathrec_gpu.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(prc_gpu_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2110_00085_b200.build import build
    return C.CDLL(build())


def test_library_exports_every_declared_entry_point(lib):
    syms = declared_symbols()
    assert len(syms) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (prc_gpu_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        getattr(lib, s)


def test_library_is_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib._name],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_paths_without_gpu(lib):
    lib.prc_gpu_last_error.restype = C.c_char_p
    p = C.c_void_p()
    rc = lib.prc_gpu_ctx_create(0, C.byref(p))
    # this container has no GPU: the library must fail loudly, never fall back
    assert rc in (abi.PRC_ERR_CUDA, abi.PRC_OK)
    if rc != abi.PRC_OK:
        assert lib.prc_gpu_last_error()
    assert lib.prc_gpu_ctx_create(0, None) == abi.PRC_ERR_INVALID
    assert lib.prc_gpu_render(None, None, None, None, None, None) == abi.PRC_ERR_INVALID
    assert lib.prc_gpu_evaluate(None, None, None, None, None) == abi.PRC_ERR_INVALID
    assert lib.prc_gpu_sort_by_size(None, None) == abi.PRC_ERR_INVALID


def test_struct_layouts_match_header(tmp_path):
    names = {"prc_scene_desc": abi.SceneDesc, "prc_species_desc": abi.SpeciesDesc,
             "prc_surface_desc": abi.SurfaceDesc, "prc_detector_desc": abi.DetectorDesc,
             "prc_light_desc": abi.LightDesc, "prc_gpu_params": abi.Params,
             "prc_gpu_render_opts": abi.RenderOpts, "prc_gpu_store_info": abi.StoreInfo,
             "prc_gpu_eval_opts": abi.EvalOpts, "prc_gpu_eval_result": abi.EvalResult,
             "prc_gpu_adam_config": abi.AdamConfig, "prc_gpu_reconstruct_opts": abi.ReconstructOpts}
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "pathrec_gpu.h"\nint main(void){\n' +
                   "".join(f'printf("%zu\\n", sizeof({n}));\n' for n in names) + "return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    sizes = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    for (n, cls), sz in zip(names.items(), sizes):
        assert C.sizeof(cls) == sz, n


def test_header_compiles_as_c_and_cpp(tmp_path):
    for comp, ext in (("gcc", "c"), ("g++", "cpp")):
        f = tmp_path / f"h.{ext}"
        f.write_text('#include "pathrec_gpu.h"\nint main(void){return PRC_OK;}\n')
        subprocess.check_call([comp, "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(f),
                               "-o", str(tmp_path / f"h_{ext}")])


def test_library_loads_before_torch():
    """The engine and torch share the soname libnccl.so.2: the engine links the NCCL torch
    ships (2.28), so loading it first must not break a later `import torch` (torch's
    libtorch_cuda needs 2.28-only symbols)."""
    import subprocess
    import sys
    code = ("import ctypes, sys; sys.path.insert(0, %r); "
            "from paper_2110_00085_b200.build import OUT; ctypes.CDLL(OUT); import torch.distributed") % ROOT
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
