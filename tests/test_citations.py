"""Every `file.hpp:L` / `file.hpp:A-B` citation in the drop-in boundary (include/*.h,
include/mpm_gpu/*.hpp) must resolve in the reference: the range lies inside the file, and when the
text just before the citation (since the previous one on the line) names reference symbols, at least
one of them occurs in the cited lines (+-2).

Runs on CPU; needs /root/reference (skipped where it is absent, e.g. on the GPU box)."""
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/proj")
CITE = re.compile(r"\b([a-z_]+\.(?:hpp|cpp))(?::(\d+)(?:-(\d+))?)((?:\s*,\s*:\d+(?:-\d+)?)*)")
IDENT = re.compile(r"[A-Za-z_][A-Za-z0-9_]{3,}")
STOP = {"const", "void", "with", "from", "this", "that", "into", "only", "line", "file", "every", "here", "same",
        "each", "none", "true", "false", "return", "struct", "template", "class", "double", "float", "size", "step",
        "int64", "int64_t", "NULL", "mpm_", "state", "scene", "grid", "time"}


def ref_path(name):
    for sub in ("include/mpm", "src", "tests", "tools"):
        p = REF / sub / name
        if p.exists():
            return p
    return None


def citing_files():
    return sorted((ROOT / "include").rglob("*.h")) + sorted((ROOT / "include").rglob("*.hpp"))


@pytest.mark.skipif(not REF.exists(), reason="/root/reference not present")
@pytest.mark.parametrize("path", citing_files(), ids=lambda p: str(p.relative_to(ROOT)))
def test_boundary_citations_resolve(path):
    bad = []
    n = 0
    for lineno, line in enumerate(path.read_text().splitlines(), 1):
        prev = 0
        for m in CITE.finditer(line):
            seg, prev = line[prev:m.start()], m.end()
            name = m.group(1)
            rp = ref_path(name)
            if rp is None:
                continue
            lines = rp.read_text().splitlines()
            ranges = [(int(m.group(2)), int(m.group(3) or m.group(2)))]
            for extra in re.findall(r":(\d+)(?:-(\d+))?", m.group(4) or ""):
                ranges.append((int(extra[0]), int(extra[1] or extra[0])))
            text = "\n".join(lines)
            names = {w for w in IDENT.findall(seg) if w not in STOP and re.search(r"\b%s\b" % re.escape(w), text)}
            for k, (a, b) in enumerate(ranges):  # a ', :L' continuation is range-checked only
                n += 1
                if not (1 <= a <= b <= len(lines)):
                    bad.append(f"{path.name}:{lineno} {name}:{a}-{b} outside the file ({len(lines)} lines)")
                    continue
                window = "\n".join(lines[max(0, a - 3):min(len(lines), b + 2)])
                if k == 0 and names and not any(re.search(r"\b%s\b" % re.escape(w), window) for w in names):
                    bad.append(f"{path.name}:{lineno} {name}:{a}-{b} does not contain any of {sorted(names)}")
    assert not bad, "\n".join(bad)
    assert n > 0 or path.suffix == ".hpp"
