"""CPU-only checks of the C ABI: the library loads, exports every symbol include/*.h declares,
the ctypes descriptor mirrors the C struct byte for byte, and host-side validation returns the
documented status codes (no compute call is made without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2404_11068_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    B.build_attn()
    from paper_2404_11068_b200 import evoattn
    return evoattn.load()


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(evo_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    names = _declared("evo_attn.h")
    assert "evo_attn_fwd" in names and "evo_attn_bwd" in names
    for n in names:
        assert hasattr(lib, n), f"libevoattn.so does not export {n}"
    assert lib.evo_abi_version() == 1


def test_dap_library_exports(tmp_path):
    if not os.path.exists(os.path.join(ROOT, "include", "evo_dap.h")):
        pytest.skip("no DAP header")
    path = B.build_dap()
    dl = ctypes.CDLL(path)
    for n in _declared("evo_dap.h"):
        assert hasattr(dl, n), f"libevodap.so does not export {n}"


def test_pair_bias_exports_and_descriptor(lib, tmp_path):
    for n in _declared("evo_pair_bias.h"):
        assert hasattr(lib, n), f"libevoattn.so does not export {n}"
    from paper_2404_11068_b200.evoattn import PairBiasDesc
    fields = [f[0] for f in PairBiasDesc._fields_]
    src = tmp_path / "pb.c"
    body = "\n".join(f'printf("{f} %zu\\n", offsetof(evo_pair_bias_desc_t, {f}));' for f in fields)
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "evo_pair_bias.h"\n'
                   'int main(void){printf("size %zu\\n", sizeof(evo_pair_bias_desc_t));' + body + "}")
    exe = tmp_path / "pb"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = dict(l.split() for l in subprocess.check_output([str(exe)]).decode().splitlines())
    assert int(out["size"]) == ctypes.sizeof(PairBiasDesc)
    for f in fields:
        assert int(out[f]) == getattr(PairBiasDesc, f).offset, f


def test_global_attn_exports_and_descriptor(lib, tmp_path):
    for n in _declared("evo_global_attn.h"):
        assert hasattr(lib, n), f"libevoattn.so does not export {n}"
    from paper_2404_11068_b200.evoattn import GlobalAttnDesc
    fields = [f[0] for f in GlobalAttnDesc._fields_]
    src = tmp_path / "ga.c"
    body = "\n".join(f'printf("{f} %zu\\n", offsetof(evo_global_attn_desc_t, {f}));' for f in fields)
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "evo_global_attn.h"\n'
                   'int main(void){printf("size %zu\\n", sizeof(evo_global_attn_desc_t));' + body + "}")
    exe = tmp_path / "ga"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = dict(l.split() for l in subprocess.check_output([str(exe)]).decode().splitlines())
    assert int(out["size"]) == ctypes.sizeof(GlobalAttnDesc)
    for f in fields:
        assert int(out[f]) == getattr(GlobalAttnDesc, f).offset, f


def test_ln_proj_exports_and_descriptor(lib, tmp_path):
    for n in _declared("evo_ln_proj.h"):
        assert hasattr(lib, n), f"libevoattn.so does not export {n}"
    from paper_2404_11068_b200.evoattn import LnProjDesc
    fields = [f[0] for f in LnProjDesc._fields_]
    src = tmp_path / "lp.c"
    body = "\n".join(f'printf("{f} %zu\\n", offsetof(evo_ln_proj_desc_t, {f}));' for f in fields)
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "evo_ln_proj.h"\n'
                   'int main(void){printf("size %zu\\n", sizeof(evo_ln_proj_desc_t));' + body + "}")
    exe = tmp_path / "lp"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = dict(l.split() for l in subprocess.check_output([str(exe)]).decode().splitlines())
    assert int(out["size"]) == ctypes.sizeof(LnProjDesc)
    for f in fields:
        assert int(out[f]) == getattr(LnProjDesc, f).offset, f


def test_ln_proj_validation(lib):
    from paper_2404_11068_b200.evoattn import LnProjDesc
    d = LnProjDesc()
    d.rows, d.C, d.N, d.eps, d.x_ld, d.out_ld = 256, 96, 512, 1e-5, 96, 512
    p = ctypes.c_void_p(16)
    lib.evo_ln_proj_fwd.restype = ctypes.c_int
    assert lib.evo_ln_proj_fwd(ctypes.byref(d), p, p, p, p, None, p, None, None, None) == 4
    d.C, d.N = 128, 100
    assert lib.evo_ln_proj_fwd(ctypes.byref(d), p, p, p, p, None, p, None, None, None) == 4
    d.N, d.x_ld = 512, 132
    assert lib.evo_ln_proj_fwd(ctypes.byref(d), p, p, p, p, None, p, None, None, None) == 3


def test_pair_bias_validation(lib):
    from paper_2404_11068_b200.evoattn import PairBiasDesc
    d = PairBiasDesc()
    d.Li, d.Lj, d.C, d.H, d.eps = 4, 4, 96, 4, 1e-5
    d.z_str = (ctypes.c_int64 * 3)(4 * 96, 96, 1)
    d.b_str = (ctypes.c_int64 * 3)(16, 4, 1)
    p = ctypes.c_void_p(16)
    lib.evo_pair_bias_fwd.restype = ctypes.c_int
    rc = lib.evo_pair_bias_fwd(ctypes.byref(d), p, p, p, p, p, p, p, None)
    assert rc == 4  # EVO_E_UNSUPPORTED (C = 96)
    d.C, d.H = 128, 5
    assert lib.evo_pair_bias_fwd(ctypes.byref(d), p, p, p, p, p, p, p, None) == 4
    d.H, d.eps = 4, 0.0
    assert lib.evo_pair_bias_fwd(ctypes.byref(d), p, p, p, p, p, p, p, None) == 1
    d.eps = 1e-5
    d.z_str = (ctypes.c_int64 * 3)(4 * 128, 128, 2)
    assert lib.evo_pair_bias_fwd(ctypes.byref(d), p, p, p, p, p, p, p, None) == 3


def test_descriptor_layout_matches_c(tmp_path):
    from paper_2404_11068_b200.evoattn import Desc
    src = tmp_path / "sz.c"
    fields = [f[0] for f in Desc._fields_]
    body = "\n".join(f'printf("{f} %zu\\n", offsetof(evo_attn_desc_t, {f}));' for f in fields)
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "evo_attn.h"\n'
                   'int main(void){printf("size %zu\\n", sizeof(evo_attn_desc_t));' + body + "}")
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = dict(l.split() for l in subprocess.check_output([str(exe)]).decode().splitlines())
    assert int(out["size"]) == ctypes.sizeof(Desc)
    for f in fields:
        assert int(out[f]) == getattr(Desc, f).offset, f


def _good_desc():
    from paper_2404_11068_b200.evoattn import Desc
    d = Desc()
    d.B, d.H, d.Lq, d.Lk, d.D, d.dtype, d.scale = 4, 2, 64, 64, 32, 0, 32 ** -0.5
    for name in ("q_str", "k_str", "v_str", "g_str", "o_str"):
        setattr(d, name, (ctypes.c_int64 * 3)(64 * 2 * 32, 32, 2 * 32))  # [B, L, H, D] storage
    d.bias_kind = 1
    d.bias_str = (ctypes.c_int64 * 4)(0, 64 * 64, 64, 1)
    d.has_mask, d.has_gate = 1, 1
    d.mask_str = (ctypes.c_int64 * 2)(64, 1)
    return d


@pytest.mark.parametrize("mutate,status", [
    (lambda d: None, 0),
    (lambda d: setattr(d, "D", 12), 4),
    (lambda d: setattr(d, "D", 128), 4),
    (lambda d: setattr(d, "dtype", 7), 1),
    (lambda d: setattr(d, "scale", 0.0), 1),
    (lambda d: setattr(d, "scale", float("nan")), 1),
    (lambda d: setattr(d, "B", -1), 2),
    (lambda d: setattr(d, "H", 0), 2),
    (lambda d: setattr(d, "Lk", 20000), 4),
    (lambda d: setattr(d, "bias_kind", 3), 1),
    (lambda d: setattr(d, "bias_str", (ctypes.c_int64 * 4)(0, 4096, 64, 2)), 4),  # no unit stride
    (lambda d: setattr(d, "bias_str", (ctypes.c_int64 * 4)(0, 4096, 1, 64)), 0),  # end-node view
    (lambda d: setattr(d, "bias_str", (ctypes.c_int64 * 4)(0, 4096, 63, 1)), 3),  # 126-B rows
    (lambda d: setattr(d, "q_str", (ctypes.c_int64 * 3)(4096, 32, 60)), 3),
    (lambda d: setattr(d, "has_gate", 2), 1),
])
def test_validation_status(lib, mutate, status):
    d = _good_desc()
    mutate(d)
    assert lib.evo_attn_validate(ctypes.byref(d)) == status, lib.evo_last_error_detail()
    if status:
        assert lib.evo_last_error_detail()  # names the offending field


def test_null_arguments_rejected_before_any_cuda_call(lib):
    d = _good_desc()
    rc = lib.evo_attn_fwd(ctypes.byref(d), None, None, None, None, None, None, None, None, None)
    assert rc == 1
    assert lib.evo_attn_fwd(None, None, None, None, None, None, None, None, None, None) == 1
    ws = lib.evo_attn_bwd_workspace_bytes(ctypes.byref(d))
    assert ws > 0
    # bwd with too small a workspace is refused without touching the device
    fake = ctypes.c_void_p(1 << 20)
    rc = lib.evo_attn_bwd(ctypes.byref(d), *([fake] * 15), ctypes.c_size_t(16), None)
    assert rc == 5, lib.evo_last_error_detail()


def test_status_strings(lib):
    names = [lib.evo_status_string(i).decode() for i in range(7)]
    assert names == ["EVO_OK", "EVO_E_INVALID", "EVO_E_SHAPE", "EVO_E_ALIGN",
                     "EVO_E_UNSUPPORTED", "EVO_E_WORKSPACE", "EVO_E_CUDA"]


def test_product_package_does_not_reference_oracle():
    """The product path never imports/links the oracle."""
    pkg = os.path.join(ROOT, "paper_2404_11068_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import oracle|from oracle)", txt, re.M), f
                assert "liboracle" not in txt and "evo_oracle" not in txt, f
