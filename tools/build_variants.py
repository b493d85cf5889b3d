"""Build libbrng variants with extra -D defines into tools/variants/ (scratch,
git-ignored) for tools/variant_time.py.

usage: python tools/build_variants.py name=DEF1,DEF2 name2=DEF3 ...
(an empty define list builds the current defaults)."""
import importlib.util
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location(
    "_b", os.path.join(ROOT, "paper_1412_4825_b200", "_build.py"))
_b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(_b)


def one(arg):
    name, _, defs = arg.partition("=")
    out = os.path.join(ROOT, "tools", "variants", name + ".so")
    _b.build(out=out, defines=tuple(d for d in defs.split(",") if d), tag=name)
    return out


if __name__ == "__main__":
    os.makedirs(os.path.join(ROOT, "tools", "variants"), exist_ok=True)
    with ThreadPoolExecutor(4) as ex:
        for o in ex.map(one, sys.argv[1:]):
            print(o)
