"""Full-size config 3 (R-MAT 2^20, Δ=32) 1-SA digests from the pruned C oracle (oracle/rowblock_oracle.c,
pinned to the reference on every golden case by tests/test_oracle.py).  The Python reference cannot
run this size; the oracle takes ~8 min per τ on one core, so the committed fixture is a
SHA-256 digest of each output array plus the input's digest (synth is deterministic across machines).

    python tests/golden/make_golden_cfg3.py 0.9,0.7

RB_GOLDEN_OUT=<file> writes elsewhere (to run several τ in parallel and merge the entries).
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2202_05868_b200 import synth  # noqa: E402

OUT = os.environ.get("RB_GOLDEN_OUT") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_cfg3_full.json")


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, np.int64)).tobytes()).hexdigest()


def main():
    taus = [float(t) for t in sys.argv[1].split(",")]
    dA, bounds, cfg, meta = synth.make("3", scale=1, device="cpu")
    rp, ci = dA.row_ptr.numpy(), dA.col_idx.numpy()
    doc = json.load(open(OUT)) if os.path.exists(OUT) else {}
    doc["input"] = {"n_rows": dA.n_rows, "nnz": dA.nnz, "row_ptr": digest(rp), "col_idx": digest(ci)}
    for tau in taus:
        r = oracle.block_1sa_arrays(rp, ci, bounds, tau=tau, pruned=True)
        doc[repr(tau)] = {"n_groups": int(r["n_groups"]),
                          **{k: digest(r[k]) for k in ("group_of", "row_perm", "group_ptr", "seed_size",
                                                       "pattern_ptr", "pattern_idx")}}
        json.dump(doc, open(OUT, "w"), indent=1, sort_keys=True)
        print("tau", tau, "groups", r["n_groups"], flush=True)


if __name__ == "__main__":
    main()
