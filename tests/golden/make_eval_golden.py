"""Golden cases for the greedy-evaluation restatement, produced by
the REFERENCE's own functions: asrkit.criterion.collapse_path,
asrkit.trainer.edit_distance and asrkit.lexicon.split_on_silence.

Run in the build container, where the reference package is importable:
    python tests/golden/make_eval_golden.py      # writes tests/golden/eval_golden.json
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("W2L_REFERENCE", "/root/reference/pkg")
sys.path.insert(0, os.path.join(REF, "src"))

import numpy as np  # noqa: E402
from asrkit.criterion import collapse_path  # noqa: E402
from asrkit.lexicon import split_on_silence  # noqa: E402
from asrkit.trainer import edit_distance  # noqa: E402


def case(rng, kind):
    n = 8
    t = int(rng.integers(1, 40))
    # runs of tokens: paths look like Viterbi paths (repeats, blanks)
    path = np.repeat(rng.integers(0, n, size=t), rng.integers(1, 4, size=t))[:60]
    ref = [int(v) for v in rng.integers(0, n, size=int(rng.integers(0, 25)))]
    blank, rep, sil = 0, 7, int(rng.integers(-1, n))   # -1: no separator
    if kind == "asg" and path[0] == rep:
        path[0] = 1
    hyp = (collapse_path(path, "ctc", blank_id=blank) if kind == "ctc"
           else collapse_path(path, "asg", rep_id=rep))
    if sil >= 0:
        rw = [tuple(g) for g in split_on_silence(ref, sil)]
        hw = [tuple(g) for g in split_on_silence(hyp, sil)]
    else:
        rw, hw = [tuple(ref)], [tuple(hyp)]
    return {"kind": kind, "path": [int(v) for v in path], "ref": ref, "blank": blank,
            "rep": rep, "silence": sil, "hyp": [int(v) for v in hyp],
            "tok_dist": edit_distance(ref, hyp), "word_dist": edit_distance(rw, hw),
            "ref_words": len(rw)}


def main():
    rng = np.random.default_rng(20260514)
    cases = [case(rng, k) for k in ("ctc", "asg") for _ in range(60)]
    with open(os.path.join(HERE, "eval_golden.json"), "w") as f:
        json.dump(cases, f)
    print(f"wrote {len(cases)} cases")


if __name__ == "__main__":
    main()
