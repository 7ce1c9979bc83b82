"""Shared test helpers (no method arithmetic)."""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_golden(name):
    """Parse tests/golden/<name>: '#' comments, section headers, whitespace rows."""
    path = os.path.join(ROOT, "tests", "golden", name)
    sections, cur = {}, None
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            toks = line.split()
            if len(toks) == 1 and toks[0][0].isalpha():
                cur = toks[0]
                sections[cur] = []
                continue
            sections[cur].append(toks)
    return sections
