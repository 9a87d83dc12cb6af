"""C-ABI library: loads without a GPU and exports every symbol include/lmgs.h declares."""

import ctypes
import re
from pathlib import Path

from paper_2503_21364_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "lmgs.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(lmgs_\w+)\s*\(", text, re.M)))


def test_header_and_binding_agree():
    assert sorted(_lib.EXPORTS) == declared_symbols()


def test_library_loads_and_exports_all_symbols():
    L = ctypes.CDLL(str(_lib.LIB_PATH))
    for sym in declared_symbols():
        assert hasattr(L, sym), sym
    assert _lib.lib().lmgs_abi_version() == _lib.ABI_VERSION


def test_struct_layouts_match_header():
    # sizes of the by-pointer structs as compiled on x86-64 / the CUDA host side
    assert ctypes.sizeof(_lib.Camera) == 8 * (9 + 3 + 3 + 6) + 8
    assert ctypes.sizeof(_lib.Gaussians) == 8 * 6 + 8 + 8 + 8 + 8  # + page_mask, shift, pad
    assert ctypes.sizeof(_lib.Settings) == 4 * 2 + 8 * 3 + 4 + 4 + 8  # + max_instances
    assert ctypes.sizeof(_lib.Frame) == 8 * 8


def test_composite_rejects_bad_order_without_gpu():
    order = (ctypes.c_int32 * 2)(0, 5)
    st = _lib.lib().lmgs_composite_blocks(None, None, None, 2, ctypes.addressof(order), 4, None,
                                          None, None, None, None)
    assert st == _lib.LMGS_ERR_INVALID
