"""The C ABI: libpcnn.so loads on a CPU box and exports exactly what
include/pcnn.h declares, with struct layouts that match the ctypes mirror."""

import ctypes
import pathlib
import re
import subprocess

import pytest

from paper_2509_22857_b200 import _lib as L

ROOT = pathlib.Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "pcnn.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pcnn_[a-z_]+)\s*\(", text)))


def test_library_loads_without_gpu():
    lib = L.lib()
    assert lib.pcnn_abi_version() == L.ABI_VERSION == 3


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 12
    lib = ctypes.CDLL(str(L.LIB_PATH))
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(L.SYMBOLS), set(names) ^ set(L.SYMBOLS)


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include "pcnn.h"\n#include <stdio.h>\n#include <stddef.h>\nint main(void){'
                   'printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(pcnn_tensor_desc), sizeof(pcnn_unit_desc),'
                   ' sizeof(pcnn_pack_desc), sizeof(pcnn_scale_op), sizeof(pcnn_factor), sizeof(pcnn_rewrite_desc),'
                   ' offsetof(pcnn_unit_desc, npad), sizeof(pcnn_plan_options),'
                   ' offsetof(pcnn_plan_options, streamk_fill), offsetof(pcnn_plan_options, debug)); return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    want = [ctypes.sizeof(L.TensorDesc), ctypes.sizeof(L.UnitDesc), ctypes.sizeof(L.PackDesc),
            ctypes.sizeof(L.ScaleOp), ctypes.sizeof(L.Factor), ctypes.sizeof(L.RewriteDesc),
            L.UnitDesc.npad.offset, ctypes.sizeof(L.PlanOptions), L.PlanOptions.streamk_fill.offset,
            L.PlanOptions.debug.offset]
    assert got == want


def test_plan_options_defaults_host_only():
    # the library fills the defaults without a device; every field is an
    # explicit plan input (no environment variables inside libpcnn)
    o = L.PlanOptions.default()
    assert o.size == ctypes.sizeof(L.PlanOptions)
    assert (o.split, o.halo_tiles, o.fuse_projection, o.streamk, o.pdl, o.graph, o.timeline) == (1,) * 7
    assert o.band_pool == 0
    assert o.flag_sync == 0 and o.debug == 0 and abs(o.streamk_fill - 0.3) < 1e-12
    assert L.PlanOptions.default(streamk=0).streamk == 0
    with pytest.raises(KeyError):
        L.PlanOptions.default(no_such_switch=1)


def test_library_reads_no_environment():
    # the only getenv-free configuration path: no PCNN_* lookups in the .so
    strings = subprocess.check_output(["strings", str(L.LIB_PATH)]).decode(errors="replace")
    assert "PCNN_" not in "".join(l for l in strings.splitlines() if l.startswith("PCNN_"))
    assert not any(l.startswith("PCNN_") for l in strings.splitlines())


def test_device_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(L.PcnnError):
        L.require_device()
    assert L.lib().pcnn_device_ok() == 0


def test_workspace_bytes_is_host_only():
    # a spatial tensor reserves the larger of its float32 blocked layout and
    # the split fp16 hi/lo layout (two planes [C/8][B][H+2][W+2][8] halves)
    split = 8 * 8 * 34 * 34
    assert split > 8 * 4 * 32 * 32
    descs = L.array(L.TensorDesc, [L.TensorDesc(c=3, h=32, w=32, cb=4, nblk=1, is_vector=0, offset=0),
                                   L.TensorDesc(c=10, h=1, w=1, cb=16, nblk=1, is_vector=1, offset=split)])
    assert L.lib().pcnn_workspace_bytes(descs, 2, 8) == 4 * (split + 8 * 16)
