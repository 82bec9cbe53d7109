"""The run-time specialised trace kernel (trace_jit.cpp, used for all-T paths) against the
generic packed kernel (PLT_TRACE_JIT=0, run in a subprocess since the switch is read once
per process): identical masks and guard-band flags, outputs equal up to float32 error
propagation -- the JIT evaluates each step's relative index eta(lambda) as a fitted
polynomial (within ~1 ulp, trace_jit.cpp fit_eta) instead of the glass formula and a
reciprocal, so the two kernels round differently (~1e-5 mm after 10 surfaces).
Both are parity-checked against the oracle elsewhere (test_gpu_trace.py runs the JIT for
all-T paths and the generic kernel for ghost paths)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from plt_inputs import configs as C
from plt_inputs import rays as R

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(os.environ.get("PLT_TRACE_JIT") == "0" or bool(os.environ.get("PLT_TRACE_X1")),
                                 reason="the process runs with the JIT kernel switched off (developer knob)")]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_jit_matches_generic_kernel(gpu_lib, tmp_path, name):
    import torch
    plt = gpu_lib
    out = tmp_path / "generic.npz"
    code = f"""
import sys; sys.path.insert(0, {ROOT!r})
import numpy as np, torch
import paper_2605_04017_b200 as plt
from plt_inputs import configs as C, rays as R
cfg = C.CONFIGS[{name!r}]
lens = plt.Lens(C.lens_text({name!r}), **cfg["opts"])
d = plt.rays_to_device(R.gen_rays(cfg["law"], 17, 0, (1 << 18) + 5))
h = plt.alloc_hits((1 << 18) + 5, flags=True)
plt.trace_rays(lens, lens.all_t_id(), d, h, direction=cfg["direction"])
torch.cuda.synchronize()
np.savez({str(out)!r}, **{{k: h[k].cpu().numpy() for k in plt.HIT_KEYS + ("mask_bits", "flags")}})
"""
    env = dict(os.environ, PLT_TRACE_JIT="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=600)
    g = np.load(out)
    cfg = C.CONFIGS[name]
    lens = plt.Lens(C.lens_text(name), **cfg["opts"])
    n = (1 << 18) + 5
    d = plt.rays_to_device(R.gen_rays(cfg["law"], 17, 0, n))
    h = plt.alloc_hits(n, flags=True)
    plt.trace_rays(lens, lens.all_t_id(), d, h, direction=cfg["direction"])
    torch.cuda.synchronize()
    assert np.array_equal(h["mask_bits"].cpu().numpy(), g["mask_bits"])
    assert np.array_equal(h["flags"].cpu().numpy(), g["flags"])
    for k, tol in (("px", 4e-5), ("py", 4e-5), ("dx", 4e-6), ("dy", 4e-6), ("dz", 4e-6), ("throughput", 2e-6)):
        assert np.max(np.abs(h[k].cpu().numpy() - g[k])) <= tol, k


def test_jit_out_of_range_wavelengths_take_the_exact_retrace(gpu_lib):
    """The JIT evaluates each step's relative index as a polynomial fitted on 378-791 nm;
    rays outside that range must be flagged for the float64 re-trace (exact glass
    formulas) and still match the oracle."""
    import oracle
    from gpu_helpers import compare_trace, gpu_trace
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    gl = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    ol = oracle.load_lens(C.lens_text("C2"), cfg["opts"])
    rays = R.gen_rays(cfg["law"], 23, 0, 1 << 16)
    lam = rays["lambda_nm"].copy()
    lam[0::3] = 350.0
    lam[1::3] = 850.0
    rays["lambda_nm"] = lam
    g = gpu_trace(plt, gl, gl.all_t_id(), rays)
    o = oracle.trace(ol, gl.all_t_id(), 0, rays, threads=oracle.host_threads())
    compare_trace(g, o)
    out = (lam < 378.0) | (lam > 791.0)
    assert np.all(g["flags"][out] == 1)


def test_trace_kernel_reports_the_kernel_that_runs(gpu_lib, tmp_path):
    """plt_trace_kernel makes the kernel choice observable (the JIT and generic kernels
    differ in the last bits): on this box all-T paths must run the run-time specialised
    kernel (NVRTC present -- so the bench and the parity tests measure the kernel DESIGN.md
    describes), ghosts the generic packed kernel, fp64 the float64 kernel; with
    PLT_TRACE_JIT=0 the all-T path reports the generic kernel."""
    plt = gpu_lib
    cfg = C.CONFIGS["C2"]
    lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
    assert plt.trace_kernel(lens, lens.all_t_id()) == "jit"
    assert plt.trace_kernel(lens, 1 << 10, precision=plt.FP64) == "fp64"
    ghost = sorted(lens.enumerate_ghosts(2)[0])[-1]
    assert plt.trace_kernel(lens, ghost) == "packed"
    code = f"""
import sys; sys.path.insert(0, {ROOT!r})
import paper_2605_04017_b200 as plt
from plt_inputs import configs as C
cfg = C.CONFIGS["C2"]
lens = plt.Lens(C.lens_text("C2"), **cfg["opts"])
print(plt.trace_kernel(lens, lens.all_t_id()))
"""
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PLT_TRACE_JIT="0"), capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("packed"), r.stdout + r.stderr
