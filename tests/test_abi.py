"""CPU-side checks of the C-ABI boundary: the library loads, exports every
entry point include/livepipe_b200.h declares, and the ctypes struct layouts
match the C compiler's."""

import ctypes
import os
import subprocess
import sys

import pytest

from paper_2512_04677_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    lib = L.load()
    syms = L.header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.lp_abi_version() == L.ABI_VERSION == 8


def test_ctypes_signatures_cover_header():
    assert set(L.header_symbols()) == set(L._SIGS)


def test_struct_layout_matches_c(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "livepipe_b200.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(lp_block_desc),"
        " sizeof(lp_rope_geom), sizeof(lp_qkv_epi), sizeof(lp_gemm_args), sizeof(lp_attn_args),"
        " offsetof(lp_block_desc, noise_key), offsetof(lp_gemm_args, qkv), sizeof(lp_conv_taps),"
        " offsetof(lp_gemm_args, conv), offsetof(lp_gemm_args, row_stats));return 0;}\n")
    exe = tmp_path / "sz"
    r = subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                       capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("no C compiler: " + r.stderr)
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = [ctypes.sizeof(L.BlockDesc), ctypes.sizeof(L.RopeGeom), ctypes.sizeof(L.QkvEpi),
            ctypes.sizeof(L.GemmArgs), ctypes.sizeof(L.AttnArgs), L.BlockDesc.noise_key.offset,
            L.GemmArgs.qkv.offset, ctypes.sizeof(L.ConvTaps), L.GemmArgs.conv.offset,
            L.GemmArgs.row_stats.offset]
    assert got == want


def test_ops_fail_loudly_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(L.LivepipeError):
        L.call("lp_init", 0)


def test_missing_library_fails_loudly(tmp_path):
    # no CPU fallback: without the CUDA library every op raises
    code = ("import paper_2512_04677_b200._lib as L\n"
            "try:\n    L.load()\nexcept ImportError as e:\n    print('IMPORTERROR', e)\n")
    env = dict(os.environ, LIVEPIPE_LIB=str(tmp_path / "missing.so"), PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT)
    assert "IMPORTERROR" in out.stdout and "no CPU fallback" in out.stdout
