"""Loader for tests/golden/*.txt fixtures (key = python literal; '#' comments carry citations)."""
import ast
import os

_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str) -> dict:
    out = {}
    with open(os.path.join(_DIR, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, v = line.split("=", 1)
            out[k.strip()] = ast.literal_eval(v.strip())
    return out
