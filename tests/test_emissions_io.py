"""W2LE emissions I/O, pinned to a file written by the reference's
own dump_emissions (tests/golden/make_w2le.py); CPU only."""
import os

import numpy as np
import pytest
import torch

from paper_1812_07625_b200 import emissions_io as eio
from paper_1812_07625_b200.errors import ContractError, EmissionsFormatError

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_reads_reference_file_bit_exact():
    e = eio.load_emissions(os.path.join(GOLDEN, "ref_emissions.w2le"))
    want = np.load(os.path.join(GOLDEN, "ref_emissions.npy"))
    assert e.dtype == np.float32 and np.array_equal(e, want)


def test_writes_reference_bytes(tmp_path):
    want = np.load(os.path.join(GOLDEN, "ref_emissions.npy"))
    p = tmp_path / "x.w2le"
    eio.dump_emissions(want, p)
    with open(p, "rb") as f, open(os.path.join(GOLDEN, "ref_emissions.w2le"), "rb") as g:
        assert f.read() == g.read()


def test_format_errors(tmp_path):
    p = tmp_path / "bad.w2le"
    p.write_bytes(b"W2LE")
    with pytest.raises(EmissionsFormatError, match="too short"):
        eio.load_emissions(p)
    p.write_bytes(b"XXXX" + b"\0" * 12)
    with pytest.raises(EmissionsFormatError, match="bad magic"):
        eio.load_emissions(p)
    good = np.ones((3, 2), np.float32)
    eio.dump_emissions(good, p)
    raw = bytearray(p.read_bytes())
    raw[4] = 2
    p.write_bytes(bytes(raw))
    with pytest.raises(EmissionsFormatError, match="unsupported version"):
        eio.load_emissions(p)
    eio.dump_emissions(good, p)
    p.write_bytes(p.read_bytes()[:-4])
    with pytest.raises(EmissionsFormatError, match="payload size mismatch"):
        eio.load_emissions(p)
    with pytest.raises(ContractError):
        eio.dump_emissions(np.ones(5, np.float32), p)
    with pytest.raises(ContractError):
        eio.dump_emissions(np.ones((0, 3), np.float32), p)


def test_batch_loader_pads_and_stacks(tmp_path):
    rng = np.random.default_rng(7)
    es = [rng.standard_normal((t, 6)).astype(np.float32) for t in (5, 9, 1)]
    paths = []
    for i, e in enumerate(es):
        paths.append(tmp_path / f"{i}.w2le")
        eio.dump_emissions(e, paths[-1])
    host, lens = eio.load_emissions_batch(paths, pin=False)
    assert host.shape == (3, 9, 6) and lens.tolist() == [5, 9, 1]
    for i, e in enumerate(es):
        assert np.array_equal(host[i, :len(e)].numpy(), e)
        assert not host[i, len(e):].any()
    eio.dump_emissions(np.ones((2, 4), np.float32), tmp_path / "n4.w2le")
    with pytest.raises(ContractError, match="disagree on N"):
        eio.load_emissions_batch([paths[0], tmp_path / "n4.w2le"], pin=False)
