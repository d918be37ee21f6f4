import os

_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str = "spec_examples.txt") -> dict:
    out = {}
    with open(os.path.join(_DIR, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, val, *_ = line.split()
            out[key] = float(val)
    return out
