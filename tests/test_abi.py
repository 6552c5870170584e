"""C-ABI boundary (CPU, no compute calls): the in-tree library loads and exports every
function declared in include/*.h; the Python binding names match; the product package
never imports the oracle."""
import ast
import ctypes
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"^\s*(?:int|int64_t|const char\*)\s+(skew_\w+)\s*\(", txt, flags=re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    from paper_1912_04062_b200 import build
    lib = build.build()
    L = ctypes.CDLL(lib)
    declared = _declared()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(L, name), name


def test_binding_covers_declarations():
    import paper_1912_04062_b200 as m
    assert _declared() == set(m.EXPORTS)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1912_04062_b200")
    for f in glob.glob(os.path.join(pkg, "**", "*.py"), recursive=True):
        tree = ast.parse(open(f).read())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                assert not any(a.name.split(".")[0] == "oracle" for a in node.names), f
            if isinstance(node, ast.ImportFrom):
                assert (node.module or "").split(".")[0] != "oracle", f
    for f in glob.glob(os.path.join(pkg, "csrc", "*")):
        assert "oracle" not in open(f).read().lower(), f


def test_no_gpu_means_loud_failure():
    import torch
    import paper_1912_04062_b200 as m
    if torch.cuda.is_available():
        return
    try:
        m.skew_eig(torch.zeros((4, 4), dtype=torch.float64))
    except RuntimeError as e:
        assert "CUDA" in str(e) or "cuda" in str(e)
    else:
        raise AssertionError("expected a loud failure without a GPU")
