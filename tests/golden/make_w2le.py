"""Writes tests/golden/ref_emissions.w2le with the REFERENCE's dump_emissions
(decoder.py:622-633) so the W2LE reader is pinned to the reference's bytes.
Run in the build container (imports /root/reference); the file is committed."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from asrkit.decoder import dump_emissions  # noqa: E402

rng = np.random.default_rng(2026)
e = rng.standard_normal((37, 29)).astype(np.float32)
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_emissions.w2le")
dump_emissions(e, out)
np.save(out.replace(".w2le", ".npy"), e)
print(out)
