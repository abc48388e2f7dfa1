"""Copy the reference's own tests into tests/ref_suite/ (git-ignored, travels to the GPU box).

Run by __graft_entry__.build() when /root/reference exists.  Files: conftest.py ->
ref_conftest.py, reference.py (the reference tests' numpy oracles), test_X.py ->
test_ref_X.py; the only rewrite is ``from conftest import`` -> ``from ref_conftest import``.
"""

from __future__ import annotations

import sys
from pathlib import Path

SRC = Path("/root/reference/pkg/tests")
DST = Path(__file__).resolve().parents[1] / "tests" / "ref_suite"


def vendor() -> int:
    if not SRC.is_dir():
        return 0
    DST.mkdir(parents=True, exist_ok=True)
    n = 0
    for src in sorted(SRC.glob("*.py")):
        if src.name == "conftest.py":
            name = "ref_conftest.py"
        elif src.name.startswith("test_"):
            name = "test_ref_" + src.name[len("test_"):]
        else:
            name = src.name
        text = src.read_text().replace("from conftest import", "from ref_conftest import")
        dst = DST / name
        if not dst.exists() or dst.read_text() != text:
            dst.write_text(text)
        n += 1
    return n


if __name__ == "__main__":
    print(f"vendored {vendor()} files into {DST}", file=sys.stderr)
