"""The boundary is a real C ABI: a plain C99 program (tests/c_api/c_api_demo.c)
compiles against include/grass.h with gcc (CPU test) and, on a GPU box, runs
the hot path through libgrass.so with closed-form checks (GPU test)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c_api", "c_api_demo.c")
LIBDIR = os.path.join(ROOT, "paper_2604_07808_b200")


def _build(out):
    cuda = "/usr/local/cuda"
    cmd = ["gcc", "-std=c99", "-Wall", "-Werror", "-O2", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(cuda, "include"), SRC, "-o", out, "-L", LIBDIR, "-lgrass",
           "-Wl,-rpath," + LIBDIR, "-L", os.path.join(cuda, "lib64"), "-lcudart", "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_header_is_c99_and_links(tmp_path):
    import paper_2604_07808_b200 as G
    G.lib()                                            # libgrass.so is built
    assert os.path.exists(_build(str(tmp_path / "c_api_demo")))


@pytest.mark.gpu
def test_c_program_runs_the_hot_path(tmp_path):
    exe = _build(str(tmp_path / "c_api_demo"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "c api demo ok" in r.stdout
