#!/usr/bin/env python
"""Dev tool: build tagged variants of the library with extra nvcc -D flags (here, on CPU),
then on the GPU box time each with the isolated prefill / decode microbench and run the
prefill parity subset against it.

  python scripts/variants.py build poly0=-DSPD_POLY_MASK=0 poly4=-DSPD_POLY_MASK=0x1111
  python scripts/variants.py run --kernel prefill --budgets 59,148 -- poly0 poly4   (GPU box)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_19867_b200 import _build  # noqa: E402


def lib_path(tag):
    return os.path.join(_build.PKG, f"libsemipd_v_{tag}.so")


def build(specs):
    import concurrent.futures as cf
    for spec in specs:
        tag, _, flags = spec.partition("=")
        flags = flags.split(",") if flags else []
        bdir = os.path.join(_build.BUILD, "v_" + tag)
        os.makedirs(bdir, exist_ok=True)

        def one(src):
            obj = os.path.join(bdir, os.path.basename(src)[:-3] + ".o")
            subprocess.check_call([_build.nvcc(), *_build.NVCC_FLAGS, *flags, "-c", src, "-o", obj],
                                  stderr=subprocess.DEVNULL)
            return obj
        with cf.ThreadPoolExecutor(8) as ex:
            objs = list(ex.map(one, _build.sources()))
        subprocess.check_call([_build.nvcc(), *_build.ARCH, "-shared", "-o", lib_path(tag), *objs])
        print("built", lib_path(tag), flags)


def run(argv):
    i = argv.index("--")  # microbench args -- variant tags
    rest, tags = argv[:i], argv[i + 1:]
    for tag in tags:
        env = dict(os.environ, SEMIPD_LIB=lib_path(tag))
        print("== variant", tag, flush=True)
        subprocess.call([sys.executable, os.path.join(ROOT, "scripts", "microbench.py"), *rest], env=env)
        if os.environ.get("VARIANT_TESTS", "1") == "1":
            subprocess.call([sys.executable, "-m", "pytest", "-x", "-q", "-k", "prefill and not mla",
                             os.path.join(ROOT, "tests", "test_gpu_parity.py")], env=env,
                            stdout=open(os.path.join(ROOT, "gpurun_out", f"var_{tag}_tests.log"), "w"))
            print("tests:", open(os.path.join(ROOT, "gpurun_out", f"var_{tag}_tests.log")).read().strip().splitlines()[-1], flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        run(sys.argv[2:])
