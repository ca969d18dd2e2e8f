"""Every evidence file the docs cite under profiles/ exists (DESIGN.md,
README.md, profiles/README.md): a measured number in the
docs always points at a committed line, log or capture."""
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAT = re.compile(r"`((?:profiles/)?r[12]_[A-Za-z0-9_{},.*\-]+\.(?:json|txt|md|csv|ncu-rep|log))`")


def _expand(name):
    m = re.search(r"\{([^}]*)\}", name)
    if not m:
        return [name]
    return [x for part in m.group(1).split(",") for x in _expand(name[:m.start()] + part + name[m.end():])]


def test_cited_profiles_exist():
    cited, missing = 0, []
    for doc in ("DESIGN.md", "README.md", "INTEGRATION.md", os.path.join("profiles", "README.md")):
        with open(os.path.join(ROOT, doc)) as f:
            text = f.read()
        for m in PAT.finditer(text):
            name = m.group(1) if m.group(1).startswith("profiles/") else "profiles/" + m.group(1)
            for p in _expand(name):
                cited += 1
                full = os.path.join(ROOT, p)
                if not (glob.glob(full) if "*" in p else os.path.exists(full)):
                    missing.append(f"{doc}: {p}")
    assert cited > 30
    assert not missing, missing
