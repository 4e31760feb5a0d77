"""Parser for the tiny text fixtures under tests/golden/ (test helper only)."""
import os
from fractions import Fraction

import lpgen

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    """Return dict: section -> list of lines (comments and blanks dropped).
    'key: value' lines become their own single-line sections."""
    secs, cur = {}, None
    with open(os.path.join(GOLDEN, name)) as f:
        for raw in f:
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            if line.endswith(":") and " " not in line:
                cur = line[:-1]
                secs[cur] = []
            elif ":" in line and not line.endswith(".") and " :- " not in line:
                k, v = line.split(":", 1)
                secs[k.strip()] = [v.strip()]
                cur = None
            else:
                secs[cur].append(line)
    return secs


def parse_rules(lines, names):
    """'h :- a, b, not c.' (AND), 'h :- a ; b.' (OR), 'h.' (fact) ->
    list of (kind, head, pos, neg) with atoms as indices into names."""
    idx = {nm: i for i, nm in enumerate(names)}
    out = []
    for ln in lines:
        ln = ln.rstrip(".")
        if ":-" not in ln:
            out.append(("AND", idx[ln.strip()], [], []))
            continue
        h, b = ln.split(":-")
        kind = "OR" if ";" in b else "AND"
        lits = [x.strip() for x in b.replace(";", ",").split(",")]
        pos = [idx[x] for x in lits if not x.startswith("not ")]
        neg = [idx[x[4:].strip()] for x in lits if x.startswith("not ")]
        out.append((kind, idx[h.strip()], pos, neg))
    return out


def to_rules(parsed, n):
    assert all(k == "AND" for k, *_ in parsed)
    return lpgen.from_lists(n, [(h, p, q) for _, h, p, q in parsed])


def matrix(lines):
    return [[Fraction(x) for x in ln.split()] for ln in lines]


def nums(line, typ=int):
    return [typ(x) for x in line[0].split()]
