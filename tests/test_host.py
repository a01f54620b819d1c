"""CPU-side checks: the C-ABI library loads and exports every declared symbol,
host-side integer prep mirrors the reference, and the product path refuses to
run without a GPU (no CPU fallback)."""

import ctypes
import os

import numpy as np
import pytest
import torch

from paper_1812_07625_b200 import _native as nat
from paper_1812_07625_b200 import criterion as C
from paper_1812_07625_b200.errors import ContractError, TargetError
from conftest import TokenTable  # noqa: E402


def test_library_exports_every_header_symbol():
    declared = nat.header_symbols()
    assert len(declared) >= 15
    lib = nat.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert set(nat.SIGNATURES) == set(declared)
    assert "sm_100a" in nat.version()


def test_library_is_sm100a_only():
    from paper_1812_07625_b200._build import LIB
    out = os.popen(f"cuobjdump -lelf {LIB} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_workspace_sizes_and_contract_codes():
    lib = nat.lib()
    assert lib.w2l_asg_workspace_bytes(64, 1600, 30, 300) > 0
    assert lib.w2l_asg_workspace_bytes(4, 100, 33, 20) == 0          # N > 32
    assert lib.w2l_ctc_workspace_bytes(4, 100, 29, 600) == 0         # 2L+1 > 1024
    assert lib.w2l_viterbi_workspace_bytes(4, 1600, 30) > 0
    # host-side contract violations return W2L_ERR_CONTRACT without touching the GPU
    rc = lib.w2l_asg_loss_grad(None, None, None, None, None, 1, 10, 40, 3, None, None, None,
                               None, None, None, 0, 0, None)
    assert rc == nat.ERR_CONTRACT
    assert lib.w2l_status_string(4).decode() == "infeasible target"
    bad = ctypes.c_int32(7)
    assert lib.w2l_status_first_error(None, 0, ctypes.byref(bad), None) == nat.OK
    assert bad.value == -1


def test_validate_target_rules():
    table = TokenTable(["a", "b", "<2>"])
    rep = table.rep_id
    assert C.validate_target([0, 0, 1], "ctc", table) == [0, 0, 1]
    assert C.validate_target([0, 0, 0], "asg", table) == [0, rep, 0]
    assert C.validate_target([0, 0, 1, 1], "asg", table) == [0, rep, 1, rep]
    with pytest.raises(TargetError):
        C.validate_target([5], "ctc", TokenTable(["a", "b"]))
    with pytest.raises(TargetError):
        C.validate_target([0, 0], "asg", TokenTable(["a", "b"]))
    with pytest.raises(ContractError):
        C.validate_target([0], "s2s", table)


def test_collapse_path_rules():
    assert C.collapse_path([0, 0, 2, 1, 1, 2], "ctc", blank_id=2) == [0, 1]
    assert C.collapse_path([2, 2, 2], "ctc", blank_id=2) == []
    rep = TokenTable(["a", "b", "<2>"]).rep_id
    assert C.collapse_path([0, 0, rep, 1], "asg", rep_id=rep) == [0, 0, 1]
    with pytest.raises(ContractError):
        C.collapse_path([rep, 0], "asg", rep_id=rep)


def test_host_shape_contracts_precede_device_work():
    with pytest.raises(ContractError):
        C.asg_loss_grad(np.zeros((3,)), [0], np.zeros((1, 1)))
    with pytest.raises(ContractError):
        C.ctc_loss_grad(np.zeros((2, 40)), [0], 39)                  # N > 32 tokens


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only behaviour")
def test_no_cpu_fallback():
    with pytest.raises(nat.NativeLibraryError):
        C.asg_loss_grad(np.zeros((2, 2)), [0], np.zeros((2, 2)))
    with pytest.raises(nat.NativeLibraryError):
        C.viterbi_batched(np.zeros((1, 2, 2), np.float32), [2])
