"""The product package never routes through the CPU oracle (test
infrastructure only: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference arm may use it) and has no CPU compute fallback:
without the CUDA library it fails loudly (tests/test_abi.py)."""

import ast
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2512_04677_b200")


def _imports(path):
    tree = ast.parse(open(path).read())
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            for a in node.names:
                yield a.name
        elif isinstance(node, ast.ImportFrom):
            yield node.module or ""


def test_package_does_not_import_the_oracle_or_the_reference():
    for name in sorted(os.listdir(PKG)):
        if not name.endswith(".py"):
            continue
        for mod in _imports(os.path.join(PKG, name)):
            assert not mod.startswith("oracle"), (name, mod)
            assert not mod.startswith("livepipe"), (name, mod)


def test_bench_uses_the_oracle_only_in_the_cpu_legs():
    src = open(os.path.join(ROOT, "bench.py")).read()
    tree = ast.parse(src)
    users = set()
    for fn in ast.walk(tree):
        if isinstance(fn, ast.FunctionDef):
            for node in ast.walk(fn):
                if isinstance(node, (ast.Import, ast.ImportFrom)):
                    mods = [a.name for a in node.names] if isinstance(node, ast.Import) else [node.module or ""]
                    if any(m.startswith("oracle") for m in mods):
                        users.add(fn.name)
    assert users <= {"cpu_baseline", "run_reference", "_cpu_worker", "_ref_worker"}, users
