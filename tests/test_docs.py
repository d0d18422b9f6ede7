"""Every file that DESIGN.md, README.md and the profile / script indexes cite in
backticks exists in the repository (the evidence they point to is committed)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DOCS = ["DESIGN.md", "README.md", "profiles/r1/SUMMARY.md", "profiles/r2/SUMMARY.md", "scripts/README.md"]
SEARCH = ["", "profiles/r1", "profiles/r2", "profiles", "scripts", "tests", "results", "paper_2107_14774_b200",
          "paper_2107_14774_b200/csrc", "studies", "examples", "include", "oracle"]
EXTERNAL = {"SPEC.md", "PAPER.md"}  # the reference (not in this repository)
PAT = re.compile(r"`([A-Za-z0-9_./{},\-]+\.(?:py|cu|cuh|h|c|sh|json|jsonl|csv|md|ncu-rep))`")


def _expand(name):
    m = re.search(r"\{([^}]*)\}", name)
    if not m:
        return [name]
    return [name[:m.start()] + x + name[m.end():] for x in m.group(1).split(",")]


def test_cited_files_exist():
    missing = []
    for doc in DOCS:
        for ref in PAT.findall(open(os.path.join(ROOT, doc)).read()):
            for name in _expand(ref):
                if name in EXTERNAL:
                    continue
                if not any(os.path.exists(os.path.join(ROOT, d, name)) for d in SEARCH):
                    missing.append((doc, name))
    assert not missing, missing
