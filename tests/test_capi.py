"""The C-ABI library loads and exports every symbol include/*.h declares.
No compute calls here (no GPU on the CPU runner)."""
import ctypes
import os
import re

import pytest

import paper_1404_1810_b200 as amqft
from paper_1404_1810_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    inc = os.path.join(ROOT, "include")
    for fn in os.listdir(inc):
        if not fn.endswith(".h"):
            continue
        text = open(os.path.join(inc, fn)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(amqft_[a-z0-9_]+)\s*\(", text):
            names.add(m.group(1))
    return sorted(names)


def test_header_declares_entry_points():
    names = declared_functions()
    for must in ("amqft_plan_create", "amqft_plan_destroy", "amqft_exec_forward",
                 "amqft_exec_inverse", "amqft_execute_host", "amqft_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_version_string():
    assert b"sm_100a" in amqft.lib().amqft_version()


def test_no_cpu_fallback_without_device():
    """Without a CUDA device plan creation must fail loudly (AMQFT_ECUDA),
    never compute on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    with pytest.raises(amqft.AmqftError) as ei:
        amqft.Plan(4, amqft.FunctionId.Cdft, 1024, 1)
    assert ei.value.status == _native.ECUDA
    import numpy as np
    with pytest.raises(amqft.AmqftError):
        amqft.execute(4, amqft.FunctionId.Cdft, 16, np.zeros(32))


def test_invalid_requests_map_to_einval():
    import torch
    if torch.cuda.is_available():
        # device present: plan creation validates before touching it
        pass
    with pytest.raises(amqft.InvalidArgument):
        amqft.Plan(0, amqft.FunctionId.Cdft, 1024, 1)
    with pytest.raises(amqft.InvalidArgument):
        amqft.Plan(1, amqft.FunctionId.Cdft, 1024, 0)


def build_shim_caller(tmpdir):
    """g++ a reference-style caller against include/amqft_b200.hpp, linked to
    the product library (no other source change: the drop-in boundary)."""
    import subprocess
    exe = os.path.join(str(tmpdir), "shim_caller")
    lib_dir = os.path.dirname(_native.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                    "-I", "/usr/local/cuda/include", os.path.join(ROOT, "tests", "native", "shim_caller.cpp"),
                    "-o", exe, "-L", lib_dir, "-lamqft_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    return exe


def test_reference_style_caller_builds_and_has_no_cpu_path(tmp_path):
    """The C++ shim compiles a reference caller unchanged; without a CUDA
    device the call fails loudly (no CPU fallback)."""
    import subprocess
    import numpy as np
    exe = build_shim_caller(tmp_path)
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present: the GPU test runs the caller")
    except ImportError:
        pass
    inp = tmp_path / "x.f64"
    np.arange(32, dtype=np.float64).tofile(inp)
    r = subprocess.run([exe, "4", "16", str(inp), str(tmp_path / "y.f64")], capture_output=True, text=True)
    assert r.returncode == 3 and "CUDA" in r.stderr, (r.returncode, r.stderr)
