"""Static checks of the separation rules: the product never imports the oracle, the oracle
never imports the product, and the seeded-input module holds no method arithmetic imports."""
import ast
import os

from conftest import ROOT


def _imports(path):
    mods = set()
    for dirpath, _, files in os.walk(path):
        for f in files:
            if not f.endswith(".py"):
                continue
            tree = ast.parse(open(os.path.join(dirpath, f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    mods.update(a.name.split(".")[0] for a in node.names)
                elif isinstance(node, ast.ImportFrom) and node.module and node.level == 0:
                    mods.add(node.module.split(".")[0])
    return mods


def test_product_does_not_import_oracle():
    assert "oracle" not in _imports(os.path.join(ROOT, "paper_1601_08179_b200"))


def test_oracle_does_not_import_product():
    m = _imports(os.path.join(ROOT, "oracle"))
    assert "paper_1601_08179_b200" not in m and "synth" not in m


def test_synth_is_independent():
    m = _imports(os.path.join(ROOT, "synth"))
    assert not ({"oracle", "paper_1601_08179_b200"} & m)


def test_csrc_has_no_oracle_reference():
    csrc = os.path.join(ROOT, "paper_1601_08179_b200", "csrc")
    for f in os.listdir(csrc):
        assert "oracle" not in open(os.path.join(csrc, f)).read().lower() or f.endswith(".md")
