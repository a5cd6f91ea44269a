"""CPU-side checks of the C-ABI library (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mbe.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2401_05039_b200 import build, load_library

    build.build()
    return load_library()


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\**\s*(mbe_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    fns = _declared_functions()
    for f in ("mbe_load_csr", "mbe_enumerate", "mbe_free", "mbe_strerror", "mbe_last_error_detail", "mbe_get_info"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    for f in _declared_functions():
        assert hasattr(lib, f), f
    out = subprocess.check_output(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2401_05039_b200",
                                                                               "libmbe.so")]).decode()
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for f in _declared_functions():
        assert f in exported, f


def test_library_is_sm100a(lib):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                                   os.path.join(ROOT, "paper_2401_05039_b200", "libmbe.so")]).decode()
    assert "sm_100a" in out


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of mbe_config / mbe_result / mbe_output / mbe_graph_info have the C sizes and offsets."""
    from paper_2401_05039_b200 import _lib as L

    prog = tmp_path / "sz.c"
    fields = {
        "mbe_config": [f for f, _ in L.mbe_config._fields_],
        "mbe_result": [f for f, _ in L.mbe_result._fields_],
        "mbe_output": [f for f, _ in L.mbe_output._fields_],
        "mbe_graph_info": [f for f, _ in L.mbe_graph_info._fields_],
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "mbe.h"', "int main(void){"]
    for s, fs in fields.items():
        lines.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for f in fs:
            lines.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));')
    lines.append("return 0;}")
    prog.write_text("\n".join(lines))
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)])
    got = dict(line.split() for line in subprocess.check_output([str(exe)]).decode().splitlines())
    for s, fs in fields.items():
        cls = getattr(L, s)
        assert int(got[s]) == ctypes.sizeof(cls), s
        for f in fs:
            assert int(got[f"{s}.{f}"]) == getattr(cls, f).offset, f"{s}.{f}"


def test_strerror_and_input_validation_without_gpu(lib):
    from paper_2401_05039_b200 import _lib as L

    assert L.mbe_strerror(L.MBE_EOVERFLOW).startswith("frame arena")
    # out-of-range column id is rejected before any device work
    with pytest.raises(L.MBEError) as e:
        L.mbe_load_csr(2, 2, np.array([0, 1, 2], dtype=np.uint64), np.array([0, 7], dtype=np.uint32))
    assert e.value.code == L.MBE_ERANGE
    assert "col 7" in L.mbe_last_error_detail()
    with pytest.raises(L.MBEError) as e:
        L.mbe_load_csr(2, 2, np.array([0, 2, 1], dtype=np.uint64), np.array([0, 1], dtype=np.uint32))
    assert e.value.code == L.MBE_EINVAL


def test_no_cpu_fallback_without_device(lib):
    """On a machine without a CUDA device, loading fails loudly (MBE_ECUDA), never computes on the CPU."""
    import torch

    from paper_2401_05039_b200 import _lib as L

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    with pytest.raises(L.MBEError) as e:
        L.mbe_load_csr(2, 2, np.array([0, 1, 2], dtype=np.uint64), np.array([0, 1], dtype=np.uint32))
    assert e.value.code == L.MBE_ECUDA


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2401_05039_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "mbea_oracle" not in txt, f


def test_format_listing_host_only_matches_oracle_text(lib):
    """mbe_format_listing is host post-processing (no device): canonical text of records given in a
    scrambled order equals the oracle's SPEC S:544 text; size query / overflow / bad record errors."""
    import ctypes

    import oracle
    from oracle import reference as R
    from paper_2401_05039_b200 import MBEError, inputs as I, make_output, mbe_format_listing

    g = I.random_bipartite(12, 9, 0.4, 77)
    recs = list(oracle.mbea_list(g))
    rng = np.random.default_rng(5)
    rng.shuffle(recs)
    n_ids = sum(len(a) + len(b) for a, b in recs)
    out, (rec_off, n1, n2, ids) = make_output(len(recs) + 3, n_ids + 7)
    o = 0
    for k, (a, b) in enumerate(recs):
        rec_off[k], n1[k], n2[k] = o, len(a), len(b)
        ids[o:o + len(a) + len(b)] = list(a) + list(b)
        o += len(a) + len(b)
    text = mbe_format_listing(out, len(recs))
    assert text == R.listing_text(recs) and text.count(b"\n") == len(recs)
    assert mbe_format_listing(out, 0) == b""
    need = ctypes.c_uint64(0)
    small = ctypes.create_string_buffer(4)
    assert lib.mbe_format_listing(ctypes.byref(out), len(recs), small, 4, ctypes.byref(need)) == -4
    assert need.value == len(text)
    rec_off[0] = n_ids + 5  # record past cap_ids
    with pytest.raises(MBEError) as e:
        mbe_format_listing(out, len(recs))
    assert e.value.code == -1
    with pytest.raises(MBEError):
        mbe_format_listing(out, len(recs) + 4)  # n_records > cap_records
