"""The C++ include-swap drop-in (include/sinkattn.hpp): it compiles against the
reference's own matrix type (when /root/reference is present) and against the Eigen-API shim, links
libsinkattn.so, and on a GPU reproduces the oracle through the reference-shaped calls."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_demo.cpp")
LIBDIR = os.path.join(ROOT, "paper_2605_08123_b200")
REF_INC = "/root/reference/proj/include"
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"


def compile_demo(out, with_reference=False):
    cmd = ["g++", "-std=c++17", "-O2", "-o", out, SRC, "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(ROOT, "oracle", "ref_shim"), "-I/usr/local/cuda/include",
           "-L" + LIBDIR, "-lsinkattn", "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath," + LIBDIR,
           "-Wl,-rpath,/usr/local/cuda/lib64"]
    if with_reference:
        cmd += ["-DWITH_REFERENCE", "-I" + REF_INC, "-I" + JSON_DIR, os.path.join(REF_INC, "..", "src", "support.cpp")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


def test_dropin_compiles_and_links_against_the_shim(tmp_path):
    compile_demo(str(tmp_path / "demo"))


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="/root/reference not present")
def test_dropin_compiles_against_the_reference_types(tmp_path):
    compile_demo(str(tmp_path / "demo_ref"), with_reference=True)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["one_reference", "direct_four_plan"])
def test_dropin_matches_oracle_on_gpu(tmp_path, mode):
    import oracle_ref
    from paper_2605_08123_b200 import configs
    cfg = configs.CONFIGS[1]
    inp = configs.make_inputs(cfg)
    exe = str(tmp_path / "demo")
    compile_demo(exe)
    fin, fout = tmp_path / "in.bin", tmp_path / "out.bin"
    with open(fin, "wb") as f:
        np.array([cfg.L, cfg.d], dtype=np.int64).tofile(f)
        for x in (inp.Q, inp.K, inp.V, inp.G):
            np.ascontiguousarray(x[0], dtype=np.float32).tofile(f)
    args = [exe, str(fin), str(fout), str(cfg.w), str(cfg.T), str(cfg.R), str(cfg.eps)]
    if mode == "direct_four_plan":
        args.append("direct")
    r = subprocess.run(args, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = np.fromfile(fout, dtype=np.float32)
    n = cfg.L * cfg.d
    ref = oracle_ref.run(cfg, inp.Q, inp.K, inp.V, inp.G, precision=64, mode=1 if mode == "direct_four_plan" else 0)
    for k, name in enumerate(("O", "dQ", "dK", "dV")):
        g = got[k * n:(k + 1) * n].astype(np.float64)
        e = np.linalg.norm(g - ref[name].reshape(-1)) / np.linalg.norm(ref[name])
        assert e < 1e-5, (name, e)
