"""Evidence integrity: every measurement file the docs cite under profiles/ exists
(README.md, profiles/README.md, tools/README.md,
tools/exp/README.md), brace lists such as r02_bench_xl_n{1,2,4}.json expanded."""

import glob
import os
import re

from conftest import ROOT

DOCS = ("DESIGN.md", "README.md", "INTEGRATION.md", "profiles/README.md", "tools/README.md",
        "tools/exp/README.md")
REF = re.compile(r"(profiles/r0[12]_[A-Za-z0-9_.{},*\-]+|r0[12]_[A-Za-z0-9_{},*\-]+\.(?:json|jsonl|txt|log|csv))")


def _expand(pattern: str) -> list:
    out, todo = [], [pattern]
    while todo:
        p = todo.pop()
        m = re.search(r"\{([^}]*)\}", p)
        if not m:
            out.append(p)
            continue
        todo += [p[:m.start()] + alt + p[m.end():] for alt in m.group(1).split(",")]
    return out


def test_cited_profiles_exist():
    missing, cited = [], 0
    for doc in DOCS:
        text = open(os.path.join(ROOT, doc)).read()
        for m in REF.finditer(text):
            ref = m.group(1).rstrip(".,)")
            ref = ref if ref.startswith("profiles/") else "profiles/" + ref
            for p in _expand(ref):
                cited += 1
                if not glob.glob(os.path.join(ROOT, p)) and not glob.glob(os.path.join(ROOT, p) + "*"):
                    missing.append((doc, p))
    assert cited > 50 and not missing, missing
