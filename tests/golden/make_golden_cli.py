"""Golden digests of the reference's own ``trace`` documents (reference pkg/src/boardbatch/cli.py
:139-166), made by running the REFERENCE's CLI in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_cli.py

For each job the reference writes its JSON trace; the fixture keeps the sha256 and length of the
file bytes (the documents are up to a few MB of `.tolist()` floats) plus the decoded step count.
tests/test_gpu_cli.py runs this repo's ``trace`` (device path) with the same arguments and requires
byte-identical files, then replays them through ``serve`` in JSON and binary wire form.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"

# (game, batch, steps, seed); the first is the reference's own test_trace_and_serve_agree case
JOBS = [
    ("connect_four", 3, 15, 9),
    ("tic_tac_toe", 5, 12, 0),
    ("go_9x9", 4, 40, 1),
    ("backgammon", 3, 30, 2),
    ("kuhn_poker", 4, 6, 5),
    ("2048", 2, 20, 7),
]


def main():
    sys.path.insert(0, REF)
    from boardbatch.cli import main as ref_main

    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        for game, n, steps, seed in JOBS:
            path = os.path.join(tmp, f"{game}.json")
            code = ref_main(["trace", "--game", game, "--batch", str(n), "--steps", str(steps),
                             "--seed", str(seed), "--out", path])
            assert code == 0, (game, code)
            data = open(path, "rb").read()
            doc = json.loads(data)
            out[f"{game}_b{n}_s{steps}_seed{seed}"] = {
                "game": game, "batch": n, "steps": steps, "seed": seed,
                "sha256": hashlib.sha256(data).hexdigest(), "nbytes": len(data),
                "observation_shape": doc["spec"]["observation_shape"],
                "final_actions": doc["steps"][-1]["actions"] if doc["steps"] else [],
            }
    with open(os.path.join(HERE, "cli_traces.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden_cli.py (reference boardbatch cli trace)",
                   "traces": out}, fh, indent=1)
    print(f"wrote {len(out)} trace digests")


if __name__ == "__main__":
    main()
