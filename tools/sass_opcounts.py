"""Static SASS evidence: per-kernel counts of the Blackwell instructions that show which
units a kernel uses (tcgen05 MMA / TMEM loads+stores / TMA bulk copies / MUFU / packed FP32
/ FP64 / atomics), read with cuobjdump from the built libplt.so and from the run-time
specialised (NVRTC) trace kernel of the C2 all-T path.  Runs on the build host (no GPU).

    python tools/sass_opcounts.py --out profiles/r02_sass_opcounts.json
"""
import argparse
import collections
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# mnemonic prefix -> what it proves
KEYS = {
    "UTCHMMA": "tcgen05.mma kind::f16 (5th-gen tensor core)",
    "UTCBAR": "tcgen05.commit -> mbarrier",
    "LDTM": "tcgen05.ld (TMEM -> registers)",
    "STTM": "tcgen05.st (registers -> TMEM)",
    "UBLKCP": "cp.async.bulk (TMA bulk copy)",
    "SYNCS": "mbarrier (transaction barriers)",
    "ELECT": "elect.sync",
    "MUFU.TANH": "MUFU tanh", "MUFU.EX2": "MUFU ex2", "MUFU.RCP": "MUFU rcp", "MUFU.RSQ": "MUFU rsqrt",
    "MUFU.RCP64H": "MUFU fp64 rcp seed", "MUFU.RSQ64H": "MUFU fp64 rsqrt seed",
    "FFMA2": "packed FP32 FMA", "FMUL2": "packed FP32 MUL", "FADD2": "packed FP32 ADD",
    "FFMA": "FP32 FMA", "FMUL": "FP32 MUL", "FADD": "FP32 ADD",
    "DFMA": "FP64 FMA", "DMUL": "FP64 MUL", "DADD": "FP64 ADD",
    "F2FP": "fp32 -> bf16x2 pack", "FHADD": "mixed bf16/fp32 add",
    "ATOMS": "shared atomics", "ATOMG": "global atomics", "RED": "global reductions",
    "MATCH": "match.any", "VOTE": "warp vote", "BAR": "barrier", "FSETP": "fp32 compare", "PLOP3": "predicate logic",
}


def sass_functions(text):
    funcs, cur = {}, None
    for line in text.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if cur and m:
            op = m.group(1)
            funcs[cur]["_total"] += 1
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    funcs[cur][k] += 1
    return funcs


def short(name):
    for pat, nice in ((r"eval_map_kernelILi(\d+)E", "eval_map_kernel<G=\\1>"), (r"refine_kernel", "refine_kernel (fp64)"),
                      (r"trace_kernel_x2ILb(\d)E", "trace_kernel_x2<asph=\\1> (packed fp32)"),
                      (r"trace_kernelI(\w)Lb(\d)ELb(\d)E", "trace_kernel<\\1,asph=\\2,\\3>"),
                      (r"splat_kernel", "splat_kernel"), (r"resolve_kernel", "resolve_kernel"),
                      (r"gen_rays_kernel", "gen_rays_kernel"), (r"\d([a-z][a-z_]*_kernel)", "\\1")):
        m = re.search(pat, name)
        if m:
            return m.expand(nice)
    return name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sass_opcounts.json"))
    a = ap.parse_args()
    import paper_2605_04017_b200 as plt
    from plt_inputs import configs as C
    lib = os.path.join(ROOT, "paper_2605_04017_b200", "libplt.so")
    res = {}
    for name, cnt in sass_functions(subprocess.check_output(["cuobjdump", "-sass", lib], text=True)).items():
        res[short(name)] = dict(cnt)
    cfg = C.CONFIGS["C2"]
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
        f.write(lens.trace_jit_cubin(lens.all_t_id()))
        f.flush()
        for name, cnt in sass_functions(subprocess.check_output(["cuobjdump", "-sass", f.name], text=True)).items():
            res["plt_trace_jit (C2 all-T, NVRTC)"] = dict(cnt)
    doc = {"source": "cuobjdump -sass of paper_2605_04017_b200/libplt.so (sm_100a) and of the NVRTC cubin "
                     "returned by plt_trace_jit_cubin for the C2 all-T path; static instruction counts",
           "legend": KEYS, "kernels": res}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    for k, v in res.items():
        print(f"{k:45s} total {v.get('_total', 0):6d}  " +
              " ".join(f"{m}={v[m]}" for m in ("UTCHMMA", "LDTM", "STTM", "UBLKCP", "MUFU.TANH", "MUFU.EX2",
                                                "FFMA2", "FMUL2", "DFMA", "MATCH") if v.get(m)))


if __name__ == "__main__":
    main()
