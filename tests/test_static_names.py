"""Every global name bench.py, __graft_entry__.py and the package load is bound
somewhere in its module (a dangling call — e.g. a helper lost between sessions —
would otherwise only surface on the GPU box, inside a try/except that reports it
as a result)."""
import ast
import builtins
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
FILES = [ROOT / "bench.py", ROOT / "__graft_entry__.py", *sorted((ROOT / "paper_1703_10119_b200").glob("*.py"))]


def _bound(tree):
    names = set(dir(builtins)) | {"__file__", "__name__", "__doc__"}
    for n in ast.walk(tree):
        if isinstance(n, (ast.FunctionDef, ast.AsyncFunctionDef, ast.ClassDef)):
            names.add(n.name)
        elif isinstance(n, ast.Import):
            names.update((a.asname or a.name).split(".")[0] for a in n.names)
        elif isinstance(n, ast.ImportFrom):
            names.update(a.asname or a.name for a in n.names)
        elif isinstance(n, ast.Name) and isinstance(n.ctx, (ast.Store, ast.Del)):
            names.add(n.id)
        elif isinstance(n, ast.ExceptHandler) and n.name:
            names.add(n.name)
        elif isinstance(n, ast.arg):
            names.add(n.arg)
    return names


@pytest.mark.parametrize("path", FILES, ids=lambda p: p.name)
def test_no_undefined_names(path):
    tree = ast.parse(path.read_text())
    bound = _bound(tree)
    missing = sorted({f"{n.id} (line {n.lineno})" for n in ast.walk(tree)
                      if isinstance(n, ast.Name) and isinstance(n.ctx, ast.Load) and n.id not in bound})
    assert not missing, missing
