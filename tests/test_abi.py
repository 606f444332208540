"""CPU checks of the boundary: libcbp.so loads and exports every symbol
declared in include/cbp.h; argument validation without a GPU; the product
package never imports the oracle and has no CPU fallback."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HDR = ROOT / "include" / "cbp.h"
PKG = ROOT / "paper_2305_05286_b200"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HDR.read_text(), flags=re.S)
    names = set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(cbp_\w+)\s*\(", text, flags=re.M))
    return sorted(n for n in names if not n.endswith("_t"))


@pytest.fixture(scope="module")
def libcbp():
    from tools.build_native import build_cbp
    build_cbp()
    return ctypes.CDLL(str(PKG / "libcbp.so"))


def test_all_declared_symbols_exported(libcbp):
    names = declared_functions()
    assert len(names) >= 12, names
    for n in names:
        assert hasattr(libcbp, n), f"{n} declared in cbp.h but not exported"


def test_python_binding_covers_abi():
    from paper_2305_05286_b200 import cbp
    assert set(declared_functions()) <= set(cbp.SIGNATURES)


def test_construct_base_matches_input_generator(libcbp):
    import numpy as np
    import inputs
    from paper_2305_05286_b200 import construct_base
    for name in ("C1", "C2", "C4"):
        spec = inputs.CONFIGS[name].spec
        a = construct_base(spec, 1).numpy()
        b, _ = inputs.config_base(name)
        assert (a == b).all()
    with pytest.raises(Exception):
        construct_base((2, 4, 8, 2, 0, 1, 1), 1)


def test_code_create_without_device_fails_cleanly(libcbp):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    from paper_2305_05286_b200 import cbp
    base = np.zeros((2, 4), np.int16)
    h = ctypes.c_void_p()
    rc = cbp.lib().cbp_code_create(base.ctypes.data, 2, 4, 4, 0, ctypes.byref(h))
    assert rc != 0 and not h.value
    assert b"device" in cbp.lib().cbp_last_error()
    rc = cbp.lib().cbp_code_create(None, 2, 4, 4, 0, ctypes.byref(h))
    assert rc == 1


def test_product_does_not_use_oracle_or_fallback():
    for f in list(PKG.rglob("*.py")) + list((PKG / "csrc").glob("*")):
        text = f.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", text, flags=re.M), f
        assert "liboracle" not in text, f
        assert "cbp_oracle" not in text, f
    # oracle sources never include product sources either
    for f in (ROOT / "oracle").glob("*.[ch]*"):
        incs = re.findall(r'^\s*#\s*include\s*[<"]([^>"]+)[>"]', f.read_text(), flags=re.M)
        assert not [i for i in incs if "csrc" in i or "cbp_internal" in i or i.endswith(".cuh") or i == "cbp.h"], f
    py = (ROOT / "oracle" / "__init__.py").read_text()
    assert not re.search(r"^\s*(from|import)\s+paper_2305_05286_b200", py, flags=re.M)
