"""The docs name only entry points / types the C ABI declares (guards INTEGRATION / DESIGN / README
against drifting from include/adapmoe.h)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_docs_reference_declared_abi():
    header = open(os.path.join(ROOT, "include", "adapmoe.h")).read()
    declared = set(re.findall(r"\b(moe_[a-z0-9_]+)\b", header))
    missing = {}
    for doc in ("INTEGRATION.md", "DESIGN.md", "README.md"):
        text = open(os.path.join(ROOT, doc)).read()
        names = set(re.findall(r"\b(moe_[a-z0-9_]+)\b", text))
        # `moe_decode_*` style wildcards and the reference's own moe_* spellings are prose, not symbols
        names = {n for n in names if not n.endswith("_") and n not in {"moe_ref", "moe_oracle"}}
        if names - declared:
            missing[doc] = sorted(names - declared)
    assert not missing, missing
