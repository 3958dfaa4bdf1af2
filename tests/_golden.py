"""Parser for tests/golden/*.txt fixtures ("key = value  # citation")."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str) -> dict:
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line or "=" not in line:
                continue
            k, v = (s.strip() for s in line.split("=", 1))
            parts = v.split()
            vals = []
            for p in parts:
                try:
                    vals.append(int(p))
                except ValueError:
                    try:
                        vals.append(float(p))
                    except ValueError:
                        vals.append(p)
            out[k] = vals[0] if len(vals) == 1 else vals
    return out


def load_rows(name: str) -> list[list[str]]:
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                rows.append(line.split())
    return rows
