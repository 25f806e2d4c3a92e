#!/usr/bin/env python3
"""Turn the C4 oracle run of scripts/c4_oracle_run.py (GPU box host) into a
compact fixture beside the reference fixtures (tests/golden/configs/c4.npz).

    python scripts/c4_fixture.py gpurun_out/c4 <x_sha256>

The C4 oracle is the reference algorithm with the exact DCT restatement of its
eigenbasis preconditioner (oracle/phaseirls_port.py, poisson="dct"), not the
unmodified reference (which cannot run at 16384²); meta.json
records that.  u is kept on the stride-32 subgrid (2 MB) instead of stride 8.
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "configs")


def main():
    prefix, sha = sys.argv[1], sys.argv[2]
    ref = np.load(f"{prefix}_fixture.npz")          # already stride-32, no K-map (computed on the box)
    meta_run = json.load(open(f"{prefix}_oracle_meta.json"))
    keep = {k: ref[k] for k in ref.files}
    np.savez_compressed(os.path.join(OUT, "c4.npz"), **keep)
    meta_path = os.path.join(OUT, "meta.json")
    meta = json.load(open(meta_path))
    meta["c4"] = dict(shape=meta_run["shape"], x_sha256=sha, seconds=meta_run["seconds"], F=meta_run["F"],
                      outer=meta_run["outer"], pcg=meta_run["pcg"], u_norm=float(ref["u_norm"]),
                      max_outer_iters=meta_run["max_outer_iters"],
                      reference=("oracle/phaseirls_port.py unwrap(poisson='dct') on the GPU box host "
                                 f"({meta_run['cpu_threads']} threads): the reference algorithm with the exact DCT "
                                 "restatement of its eigenbasis preconditioner; the unmodified reference cannot run "
                                 "at 16384^2 (SURVEY.md §8(c))"))
    with open(meta_path, "w") as fh:
        json.dump(meta, fh, indent=1)
    print(os.path.getsize(os.path.join(OUT, "c4.npz")), "bytes")


if __name__ == "__main__":
    main()
