"""The C-ABI library builds for sm_100a, loads, and exports every symbol the public
header include/ttsw_capi.h declares (no GPU needed: nothing is called)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ttsw_capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ttsw_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_2408_03483_b200 import capi

    lib = ctypes.CDLL(capi.LIB_PATH)
    names = header_functions()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(capi.EXPORTS) == names


def test_library_is_sm100a_only():
    from paper_2408_03483_b200 import capi

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_context_creation_fails_loudly_without_gpu():
    """No CPU fallback: without a usable GPU the context reports a CUDA error."""
    import pytest

    from paper_2408_03483_b200 import capi

    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(capi.TTSWError):
        capi.Context(0)
