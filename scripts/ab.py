"""A/B builds of the CUDA library with extra -D flags, for same-box comparisons.

  python scripts/ab.py build NAME "-DPDD_FOO=1 -DPDD_BAR=2" [NAME2 "..."]
      compiles kernels.cu (the unit that instantiates the frame kernels) with
      the flags and links scripts/bin/lib_NAME.so from it and the other
      objects of the normal build (build/csrc).  scripts/bin/ is git-ignored
      and travels to the GPU box.
  python scripts/ab.py run CONFIG ITERS NAME [NAME2 ...]     (on the GPU box)
      runs scripts/prof_frame.py CONFIG ITERS once per library (PDD_LIB) and
      prints one line per variant; "base" is the in-tree library.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
BIN = os.path.join(ROOT, "scripts", "bin")
UNITS = ("kernels.cu",)


def build(pairs):
    from paper_2011_00162_b200 import build as B

    B.build()
    os.makedirs(BIN, exist_ok=True)
    objs = [os.path.join(B.BUILD, os.path.basename(s) + ".o") for s in B._sources()]
    def one(pair):
        name, flags = pair
        vobjs = list(objs)
        for u in UNITS:
            src = os.path.join(B.CSRC, u)
            obj = os.path.join(BIN, f"{name}_{u}.o")
            cmd = [B.NVCC, *B.ARCH, *B.FLAGS, *flags.split(), "-Xptxas", "-v", "-c", src, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise SystemExit(f"{name}: nvcc failed\n{r.stderr}")
            with open(os.path.join(BIN, f"{name}_ptxas.log"), "w") as f:
                f.write(r.stderr)
            vobjs[objs.index(os.path.join(B.BUILD, u + ".o"))] = obj
        lib = os.path.join(BIN, f"lib_{name}.so")
        subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *vobjs, "-ldl", "-lpthread"], check=True)
        print("built", lib, flush=True)

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=6) as ex:
        list(ex.map(one, pairs))


def run(config, iters, names):
    for n in names:
        env = dict(os.environ)
        if n != "base":
            env["PDD_LIB"] = os.path.join(BIN, f"lib_{n}.so")
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "prof_frame.py"), config, iters],
                           env=env, capture_output=True, text=True)
        out = (r.stdout.strip().splitlines() or ["<no output>"])[-1]
        print(f"{n:>16}: {out}" + ("" if r.returncode == 0 else f"  [rc {r.returncode}] {r.stderr[-400:]}"), flush=True)
        for ln in [x for x in r.stderr.splitlines() if x.startswith("PDD_PHASE")][-3:]:
            print(" " * 18 + ln, flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        a = sys.argv[2:]
        build(list(zip(a[0::2], a[1::2])))
    else:
        run(sys.argv[2], sys.argv[3], sys.argv[4:])
