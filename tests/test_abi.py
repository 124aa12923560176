"""C-ABI library contract checks that need no GPU: the library loads, exports
every symbol include/spk.h declares, and validates arguments on the host
before any launch (a failed validation returns a status and launches nothing)."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2301_13659_b200 import spk

HEADER = Path(__file__).resolve().parent.parent / "include" / "spk.h"


def declared():
    return re.findall(r"^SPK_API [^(]*?\b(spk_\w+)\(", HEADER.read_text(), flags=re.M)


def test_library_exports_every_declared_symbol():
    names = declared()
    assert len(names) >= 20
    L = spk.lib()
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(spk.EXPORTS)


def test_abi_version_matches_header():
    v = int(re.search(r"#define SPK_ABI_VERSION (\d+)", HEADER.read_text()).group(1))
    assert spk.lib().spk_abi_version() == v


def test_workspace_queries():
    g = spk.ConvGeom(1024, 15, 250, 4, 4, 200, 5, 5, 1, 1, 2, 2)
    ws = spk.conv_workspace(g, "exact")
    # 2 N-tiles of 112 maps x ceil(6250/64)=98 stages x 3 digit planes x 64 bytes + 256
    assert ws == 256 + 2 * 98 * 3 * 112 * 64
    assert spk.conv_workspace(g, "fp32") == 0
    g30 = spk.ConvGeom(256, 30, 64, 80, 125, 128, 3, 3, 1, 1, 1, 1)
    assert spk.conv_workspace(g30, "exact") > 0
    g40 = spk.ConvGeom(2, 40, 4, 8, 8, 8, 3, 3, 1, 1, 1, 1)  # T > 32: tensor path unsupported
    assert spk.conv_workspace(g40, "exact") == 0
    assert spk.stdp_workspace(g, 8) >= 4 * 200 * 1024 * 8


def _status(name, *args):
    return getattr(spk.lib(), name)(*args)


def test_host_validation_before_launch():
    L = spk.lib()
    NULL = None
    dummy = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    g = spk.ConvGeom(1, 15, 2, 5, 5, 4, 7, 7, 1, 1, 0, 0)  # kernel larger than input -> SHAPE
    assert L.spk_conv(dummy, dummy, ctypes.byref(g), 1, 1, 1.0, 1.0, dummy, NULL, dummy, 1 << 20, NULL) == 2
    assert b"Eq. 2" in L.spk_last_error()
    g = spk.ConvGeom(1, 300, 2, 5, 5, 4, 3, 3, 1, 1, 1, 1)  # T > 254
    assert L.spk_conv(dummy, dummy, ctypes.byref(g), 1, 1, 1.0, 1.0, dummy, NULL, dummy, 1 << 20, NULL) == 3
    g = spk.ConvGeom(1, 15, 2, 5, 5, 4, 3, 3, 1, 1, 1, 1)
    assert L.spk_conv(NULL, dummy, ctypes.byref(g), 1, 1, 1.0, 1.0, dummy, NULL, dummy, 1 << 20, NULL) == 1
    assert L.spk_conv(dummy, dummy, ctypes.byref(g), 1, 1, -1.0, 1.0, dummy, NULL, dummy, 1 << 20, NULL) == 1
    assert L.spk_conv(dummy, dummy, ctypes.byref(g), 1, 1, 1.0, 0.0, dummy, NULL, dummy, 1 << 20, NULL) == 1
    assert L.spk_conv(dummy, dummy, ctypes.byref(g), 1, 1, 1.0, 1.0, dummy, NULL, dummy, 8, NULL) == 4
    assert L.spk_rank_code(dummy, 1, 10, 300, 0.0, 1, dummy, NULL, 0, NULL) == 3
    assert L.spk_rank_code(NULL, 1, 10, 15, 0.0, 1, dummy, NULL, 0, NULL) == 1
    sig = (ctypes.c_double * 2)(1.0, -2.0)
    assert L.spk_dog(dummy, 1, 1, 8, 8, sig, 1, 3, 3, dummy, NULL) == 1
    sig = (ctypes.c_double * 2)(1.0, 2.0)
    assert L.spk_dog(dummy, 1, 1, 2, 2, sig, 1, 3, 0, dummy, NULL) == 2  # Eq. 1 output empty
    assert L.spk_wta(dummy, dummy, 1, 2, 4, 4, 15, 0, 1, dummy, dummy, NULL) == 1
    bad = spk.stdp_configs([(0.1, -0.1, 1.0, 0.5, 1)])  # L >= U
    g = spk.ConvGeom(1, 15, 2, 5, 5, 4, 3, 3, 1, 1, 1, 1)
    assert L.spk_stdp(dummy, ctypes.byref(g), dummy, dummy, dummy, 2, bad, 1, dummy, 1 << 20, NULL) == 1
    good = spk.stdp_configs([(0.1, -0.1, 0.0, 1.0, 1)])
    assert L.spk_stdp(dummy, ctypes.byref(g), dummy, dummy, dummy, 2, good, 1, dummy, 4, NULL) == 4
    pg = spk.PoolGeom(5, 5, 1, 1, 0, 0)
    assert L.spk_pool(dummy, 1, 1, 3, 3, 15, ctypes.byref(pg), dummy, NULL) == 2
    assert L.spk_winners_rebase(dummy, dummy, 4, 5, -1, NULL) == 1   # negative base
    assert L.spk_winners_rebase(NULL, dummy, 4, 5, 0, NULL) == 1
    assert L.spk_inhibit(dummy, dummy, 1, 2, 3, 3, 300, NULL) == 3    # T > 254
    assert L.spk_wta(dummy, dummy, 1, 2, 4, 4, 15, 65, 1, dummy, dummy, NULL) == 1  # k > 64
    assert L.spk_gather(dummy, 10, 0, dummy, NULL) == 3               # T < 1


def test_binding_refuses_cpu_tensors():
    import torch

    with pytest.raises(spk.SpkError):
        spk.gather(torch.zeros(4, dtype=torch.uint8), 15, out=torch.zeros(4))
