"""The boundary is a plain C ABI: a C99 program (no Python, no torch) includes plt.h, links
libplt.so and uses the host entry points -- lens parsing, paraxial data, ghost
enumeration with the two-call pattern -- and gets the error contract for a device call
without a GPU (or runs it when one is present)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2605_04017_b200")

C_SRC = r"""
#include <stdio.h>
#include <string.h>
#include "plt.h"
int main(void) {
    const char* text = "name dgauss\n29.475 3.76 abbe:1.670,47.1 25.2\n84.83 0.12 air 25.2\n"
                       "19.275 4.025 abbe:1.670,47.1 23.0\n40.77 3.275 abbe:1.699,30.1 23.0\n"
                       "12.75 5.705 air 18.0\n0 4.5 stop 17.1\n-14.495 1.18 abbe:1.603,38.0 17.0\n"
                       "40.77 6.065 abbe:1.658,57.3 20.0\n-20.385 0.19 air 20.0\n437.065 3.22 abbe:1.717,48.0 20.0\n"
                       "-39.73 0.0 air 20.0\n";
    plt_lens* lens = NULL;
    if (plt_lens_load(text, strlen(text), NULL, &lens) != PLT_OK) { printf("load failed: %s\n", plt_last_error()); return 1; }
    int n_opt = 0, stop = 0; double abcd[4], efl = 0, bfl = 0, sz = 0;
    if (plt_lens_info(lens, 587.5618, &n_opt, &stop, abcd, &efl, &bfl, &sz) != PLT_OK) return 2;
    int count = 0;
    if (plt_enumerate_ghosts(lens, 2, 0.0, NULL, NULL, 0, &count) != PLT_E_CAPACITY) return 3;
    uint64_t ids[64];
    if (count > 64 || plt_enumerate_ghosts(lens, 2, 0.0, ids, NULL, 64, &count) != PLT_OK) return 4;
    printf("%s|%d|%d|%.6f|%d|%llu\n", plt_version(), n_opt, stop, efl, count, (unsigned long long)ids[0]);
    plt_lens_free(lens);
    return 0;
}
"""


def test_c_program_uses_the_abi(tmp_path):
    lib = os.path.join(PKG, "libplt.so")
    if not os.path.exists(lib):
        pytest.skip("libplt.so not built")
    src = tmp_path / "consumer.c"
    src.write_text(C_SRC)
    exe = tmp_path / "consumer"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", f"-I{os.path.join(ROOT, 'include')}", str(src), "-o", str(exe),
                    f"-L{PKG}", "-lplt", f"-Wl,-rpath,{PKG}"], check=True, timeout=120)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    ver, n_opt, stop, efl, count, first = out.stdout.strip().split("|")
    assert "sm_100a" in ver and int(n_opt) == 10 and int(stop) == 5
    assert abs(float(efl) - 50.358) < 0.01                  # Kolb dGauss EFL (O13 pins)
    assert int(count) == 46 and int(first) == 1 << 10     # all-T id first, then the 45 ghosts
