"""The C ABI as a C program sees it: include/springsim_b200.h compiles as
C11 with warnings on, the in-tree library links, and a host-only call path
(argument validation, the error string, page-locked buffers) runs without a
GPU -- what a C/C++ host application embedding the engine starts from
(INTEGRATION.md §2)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2207_09334_b200")

SRC = r"""
#include <stdio.h>
#include <string.h>
#include "springsim_b200.h"
int main(void) {
    ss_scene_desc d;
    memset(&d, 0, sizeof d);
    ss_engine *e = NULL;
    int rc = ss_create(&d, &e);                   /* no masses: SS_EINVAL before any CUDA call */
    printf("%d %d|%s\n", ss_abi_version(), rc, ss_last_error());
    char *txt = NULL;
    int64_t n = 0;
    double v[3] = {0.1, 1e-05, 1e16};
    rc = ss_doc_repr(3, v, &txt, &n);             /* Python float repr, host code */
    printf("%d|%.*s", rc, (int)n, txt);
    ss_doc_free_text(txt);
    return 0;
}
"""


@pytest.mark.skipif(shutil.which("gcc") is None, reason="no C compiler")
def test_header_compiles_links_and_runs(tmp_path):
    src = tmp_path / "t.c"
    src.write_text(SRC)
    exe = tmp_path / "t"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"), str(src),
                    "-L", LIBDIR, "-lspringsim_b200", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    head, rest = out.split("\n", 1)
    assert head.startswith("2 1|") and "no masses" in head
    assert rest == "0|0.1\n1e-05\n1e+16\n"
