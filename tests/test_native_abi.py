"""CPU checks of the C-ABI library: it is built, loads, and exports every symbol
include/beast_b200.h declares (no compute calls -- there is no GPU here)."""
import ctypes
import os
import re

import pytest

from conftest import REPO


def _declared_symbols():
    with open(os.path.join(REPO, "include", "beast_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:[\w\*]+\s+\**)+(bp_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1910_03552_b200 import build

    return build.build()


def test_header_declares_entry_points():
    syms = _declared_symbols()
    assert "bp_vtrace_from_logits_f32" in syms
    assert "bp_learner_loss_f32" in syms
    assert len(syms) >= 9


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    missing = [s for s in _declared_symbols() if not hasattr(lib, s)]
    assert not missing, f"symbols declared in beast_b200.h but not exported: {missing}"


def test_python_binding_types_every_symbol(lib_path):
    from paper_1910_03552_b200 import _native

    assert set(_declared_symbols()) == set(_native.SIGNATURES)
    lib = _native.load(lib_path)
    assert lib.bp_abi_version() == 1
    # host-only helpers can be called without a GPU
    assert lib.bp_learner_loss_workspace_bytes(80, 4096, 18) > 256
    assert lib.bp_sumsq_workspace_bytes(1 << 20) > 256


def test_ops_fail_loudly_without_gpu(lib_path):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1910_03552_b200 import vtrace
    from paper_1910_03552_b200.errors import NativeError

    z = torch.zeros(2, 1)
    with pytest.raises(NativeError):
        vtrace.from_importance_weights(z, z, z, z, torch.zeros(1))


def test_host_wait_seq_without_gpu(lib_path):
    """bp_host_wait_seq (the learner's stats wait) is host-only: reached / wrap-around / timeout."""
    from paper_1910_03552_b200 import _native

    lib = _native.load(lib_path)
    word = ctypes.c_uint32(7)
    addr = ctypes.addressof(word)
    assert lib.bp_host_wait_seq(addr, 7, 1000) == 0      # reached
    assert lib.bp_host_wait_seq(addr, 5, 1000) == 0      # already past
    assert lib.bp_host_wait_seq(addr, 8, 2000) == 1      # not yet: times out
    word.value = 2                                       # wrapped past 2^32
    assert lib.bp_host_wait_seq(addr, 0xFFFFFFFE, 1000) == 0
