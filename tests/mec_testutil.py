"""Shared helpers for the test-suite (golden-file readers)."""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def golden(name: str) -> str:
    return os.path.join(ROOT, "tests", "golden", name)


def read_kv(name: str) -> dict:
    """Parse a `key v1 v2 ...` golden file (comments start with #)."""
    out = {}
    with open(golden(name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            k, *v = line.split()
            out[k] = [int(x) for x in v] if len(v) > 1 else int(v[0])
    return out
