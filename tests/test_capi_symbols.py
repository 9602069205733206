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


def test_cpp_adapter_compiles_and_links(tmp_path):
    """include/ttsw/cuda_rep.hpp (the C++ Rep drop-in) compiles against the C ABI and links."""
    src = tmp_path / "a.cpp"
    src.write_text(
        '#include "ttsw/cuda_rep.hpp"\n#include <cstdio>\n'
        "struct M { long r, c; std::vector<double> a; long rows() const {return r;} long cols() const {return c;}\n"
        "  const double* data() const {return a.data();}\n"
        "  double operator()(long i,long j) const {return a[i+j*r];} double& operator()(long i,long j){return a[i+j*r];}\n"
        "  M(long r_, long c_):r(r_),c(c_),a(r_*c_){} };\n"
        "int main(int argc, char**) { if (argc > 5) { using R = ttsw_cuda::CudaTTRep;\n"
        "  auto x = R::from_cores(1, 1, 1, nullptr, nullptr); M m(1,1); auto y = R::lin(ttsw_cuda::Axis::X, m, x);\n"
        "  auto d = R::dense<M>(y); auto z = R::axpy(1.0, x, 2.0, y, 1e-10);\n"
        "  auto w = R::compress(m, 1e-8); (void)d; (void)z; (void)w; }\n"
        '  std::puts("ok"); }\n')
    lib = os.path.join(ROOT, "paper_2408_03483_b200")
    exe = tmp_path / "a.out"
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-I" + os.path.join(ROOT, "include"), str(src), "-L" + lib,
                    "-lttsw_cuda", "-Wl,-rpath," + lib, "-o", str(exe)], check=True)
    env = dict(os.environ, LD_LIBRARY_PATH="/usr/local/cuda/lib64:" + os.environ.get("LD_LIBRARY_PATH", ""))
    assert subprocess.run([str(exe)], capture_output=True, text=True, env=env).stdout.strip() == "ok"
