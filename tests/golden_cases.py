"""Loader for the committed golden scheduling fixtures (made by the reference)."""

import gzip
import json
from functools import lru_cache
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden" / "sched_golden.json.gz"


@lru_cache(maxsize=1)
def load_cases():
    with gzip.open(GOLDEN, "rt") as fh:
        return json.load(fh)["cases"]


def oracle_tasks(case):
    return [{"id": t["id"], "period": t["period"], "deadline": t["deadline"], "hp": t["hp"],
             "stages": [(float(n), int(w)) for n, w in t["stages"]], "batch": t["batch"],
             "curve": None if t["curve"] is None else (t["curve"][0], t["curve"][1])}
            for t in case["tasks"]]


def case_ids():
    return [c["name"] for c in load_cases()]


def case_by_name(name):
    return next(c for c in load_cases() if c["name"] == name)
