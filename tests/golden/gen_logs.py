"""Generates tests/golden/search_logs.json: the reference's search log
(SearchOutcome::log, planner.hpp:95-107; CLI search_log.ndjson body,
cli.cpp:234-249) for every case of search_cases.json, pinned as an entry
count, a SHA-256 over the entries and the first entries verbatim, plus the
InfeasibleError reason list (planner.cpp:666-678) of infeasible cases.
Produced by the compiled, unmodified reference (oracle/_ref). Run in the
build container:

    make -C oracle ref && python tests/golden/gen_logs.py
"""
from __future__ import annotations

import hashlib
import json
import os
import struct
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402


def time_bits(t: float) -> str:
    return "%016x" % struct.unpack("<Q", struct.pack("<d", t))[0]


def digest(entries) -> str:
    """entries: iterable of (candidate, time_bits, reason)."""
    h = hashlib.sha256()
    for c, b, r in entries:
        h.update(f"{c}\t{b}\t{r}\n".encode())
    return h.hexdigest()


def c3_default():
    """C3 (Llama-140B, 768 devices) default mode: 218,703 log entries."""
    from paper_2405_16256_b200 import configs
    r = ref.search(configs.config("C3", full=False), jobs=16, want_log=True)
    ents = [(e["candidate"], e["time_bits"], e["reason"]) for e in r["log"]]
    rec = {"name": "C3-default", "n": len(ents), "sha256": digest(ents), "head": ents[:4],
           "candidates_simulated": r["candidates_simulated"], "candidates_pruned": r["candidates_pruned"],
           "generator": "tests/golden/gen_logs.py --c3"}
    with open(os.path.join(HERE, "c3_default_log.json"), "w") as f:
        json.dump(rec, f, indent=1)


def main():
    if "--c3" in sys.argv:
        return c3_default()
    with open(os.path.join(HERE, "search_cases.json")) as f:
        cases = json.load(f)
    out = []
    for case in cases:
        r = ref.search(case["docs"], jobs=8, want_log=True)
        rec = {"name": case["name"], "status": r["status"]}
        if r["status"] == 0:
            ents = [(e["candidate"], e["time_bits"], e["reason"]) for e in r["log"]]
            rec.update({"n": len(ents), "sha256": digest(ents), "head": ents[:4]})
        elif r["status"] == 2:
            rec["reasons"] = r.get("reasons", [])
        out.append(rec)
        print(rec["name"], rec.get("n"), file=sys.stderr)
    with open(os.path.join(HERE, "search_logs.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))


if __name__ == "__main__":
    main()
