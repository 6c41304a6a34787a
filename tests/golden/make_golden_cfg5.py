"""Full-size config 5 (262,144², 64² planted blocks at 1 % block density, rows scrambled, Δ=64, τ=0.7)
1-SA and VBR-structure digests from the C oracle (oracle/rowblock_oracle.c, pinned to the reference on
every golden case by tests/test_oracle.py; the ¼- and 1/32-scale versions are reference-generated
fixtures).  The full matrix has 687 M nonzeros: the Python reference needs a large-RAM host for it
(SURVEY §8(c)), so the committed fixture is a SHA-256 digest of each output array plus the input's
digest (synth is deterministic across machines).

    python tests/golden/make_golden_cfg5.py
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2202_05868_b200 import synth  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_cfg5_full.json")


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, np.int64)).tobytes()).hexdigest()


def main():
    t0 = time.time()
    rp, ci, vals, bounds, cfg = synth.make_host("5", scale=1)
    t1 = time.time()
    r = oracle.block_1sa_arrays(rp, ci, bounds, tau=cfg.tau)
    t2 = time.time()
    bp, bc = oracle.vbr_blocks(rp, ci, bounds, r["row_perm"], r["group_ptr"])
    t3 = time.time()
    doc = {"input": {"n_rows": len(rp) - 1, "nnz": int(rp[-1]), "row_ptr": digest(rp), "col_idx": digest(ci),
                     "values": hashlib.sha256(np.ascontiguousarray(vals).tobytes()).hexdigest()},
           "tau": cfg.tau, "n_groups": int(r["n_groups"]), "n_blocks": int(len(bc)),
           **{k: digest(r[k]) for k in ("group_of", "row_perm", "group_ptr", "seed_size", "pattern_ptr",
                                        "pattern_idx")},
           "blk_ptr": digest(bp), "blk_col": digest(bc),
           "seconds": {"synth_host": round(t1 - t0, 1), "oracle_1sa": round(t2 - t1, 1),
                       "oracle_vbr_blocks": round(t3 - t2, 1)}}
    json.dump(doc, open(OUT, "w"), indent=1, sort_keys=True)
    print(json.dumps(doc["seconds"]), "groups", doc["n_groups"], "blocks", doc["n_blocks"])


if __name__ == "__main__":
    main()
