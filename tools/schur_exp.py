"""Timing experiments on kernel K4 (k_schur): build variants here (`build`), time them on the GPU
box (`run`).  Variants differ only by -D flags (SCHUR_EXP bits in csrc/schur.cu: 1 = no epilogue,
2 = no fold and no epilogue), so their numbers bound what each phase costs.  Results of a variant
with SCHUR_EXP != 0 are wrong by construction: timing only, never a bench value."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "exp")


def variants():
    spec = os.environ.get("EXP_VARIANTS", "base:;noepi:SCHUR_EXP=1;nofold:SCHUR_EXP=2")
    out = []
    for v in spec.split(";"):
        name, _, defs = v.partition(":")
        out.append((name, [d for d in defs.split(",") if d]))
    return out


def build():
    from paper_1411_3769_b200 import build as b
    os.makedirs(OUT, exist_ok=True)
    for name, defs in variants():
        b.build(out=os.path.join(OUT, f"libpolya_{name}.so"), defines=defs, verbose=True)


def run(config="4", steps=5, warmup=2):
    res = {}
    for name, _ in variants():
        env = dict(os.environ, POLYA_LIB=os.path.join(OUT, f"libpolya_{name}.so"))
        p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--steps", str(steps),
                            "--warmup", str(warmup), "--no-e2e", "--no-cpu-baseline", "--no-ipm"],
                           env=env, capture_output=True, text=True)
        try:
            d = json.loads(p.stdout.strip().splitlines()[-1])
            res[name] = {"tflops_assembly": d["tflops_schur_assembly_only"], "ms": d["breakdown_ms"]["schur_assembly"]}
        except Exception:
            res[name] = {"error": (p.stderr or p.stdout)[-800:]}
        print(name, res[name], flush=True)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        cfg = sys.argv[2] if len(sys.argv) > 2 else "4"
        print(json.dumps(run(cfg)))
