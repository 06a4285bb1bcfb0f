"""The CPU oracle's answers at the BASELINE sizes where the oracle takes
minutes (n = 65536: ~9 min per ASPOT prefix on 16 cores), committed as
tests/golden/headline.json by tests/golden/make_headline_golden.py (the
oracle itself, run once). A GPU test reads the fixture by default and runs the
live oracle instead when $POTGPU_LIVE_ORACLE=1. Every entry carries a digest of
its instance, so a changed recipe fails loudly instead of comparing against a
stale answer."""
import hashlib
import json
import os
from types import SimpleNamespace

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "headline.json")


def live() -> bool:
    return os.environ.get("POTGPU_LIVE_ORACLE", "0") == "1"


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()[:16]


def load(name: str, *instance_arrays):
    """The golden entry `name` as an oracle-result-like object (iterations,
    status, cost, phi, gamma, tolerance, log, trace, scale)."""
    with open(PATH) as f:
        e = json.load(f)[name]
    assert e["digest"] == digest(*instance_arrays), f"golden {name}: the instance recipe changed, regenerate the fixture"
    e = dict(e)
    e["log"] = np.asarray(e["log"], dtype=np.float64).reshape(-1, 9)
    e["trace"] = np.asarray(e["trace"], dtype=np.float64)
    return SimpleNamespace(**e)
