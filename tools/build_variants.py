"""Build experiment variants of the library: python tools/build_variants.py NAME=-DX=1,-DY=2 ...

Each variant goes to variants/lib_NAME.so (objects in variants/obj_NAME; git-ignored, travels with gpurun); load
one with SYLFEM_B200_LIB=variants/lib_NAME.so.
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_01173_b200 import build as B  # noqa: E402

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(spec):
    name, _, defs = spec.partition("=")
    defines = tuple(d for d in defs.split(",") if d)
    lib = os.path.join(root, "variants", f"lib_{name}.so")
    B.build(lib=lib, obj=os.path.join(root, "variants", f"obj_{name}"), defines=defines)
    return lib


with ThreadPoolExecutor(max_workers=4) as pool:
    for lib in pool.map(one, sys.argv[1:]):
        print("built", lib)
