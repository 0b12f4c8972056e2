"""The C ABI as a reference-side binding sees it.

* Every prototype in include/qqq_b200.h has exactly the parameter types that
  `_lib.SIGNATURES` (the ctypes binding) declares, position by position.
* The ctypes snippet in INTEGRATION.md binds the same argtypes as the header.
* A plain C program (tests/c/gemm_caller.c) compiles with gcc against the
  header and links against libqqq_b200.so (CPU); on a B200 it runs one
  per-group linear through qqq_act_quant_ex -> qqq_repack_weights ->
  qqq_w4a8_gemm_pg and its y / acc are bit-identical to the oracle (GPU).
"""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qqq_b200.h")
INTEGRATION = os.path.join(ROOT, "INTEGRATION.md")
CALLER = os.path.join(ROOT, "tests", "c", "gemm_caller.c")
LIBDIR = os.path.join(ROOT, "paper_2406_09904_b200", "lib")
CUDA = "/usr/local/cuda"


def _prototypes():
    """name -> [parameter type strings] for every qqq_* prototype of the header."""
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    out = {}
    for m in re.finditer(r"^\s*(?:int|size_t|const char\*)\s+(qqq_\w+)\s*\(([^)]*)\)\s*;", src, flags=re.M):
        params = " ".join(m.group(2).split())
        types = []
        if params and params != "void":
            for p in params.split(","):
                p = p.strip()
                name = re.search(r"(\w+)$", p).group(1)
                types.append(p[: len(p) - len(name)].strip())
        out[m.group(1)] = types
    return out


def _ctype_of(c_type: str):
    from paper_2406_09904_b200 import _lib

    if c_type.endswith("*") and "qqq_gemm_config" in c_type:
        return ctypes.POINTER(_lib.GemmConfig)
    if c_type.endswith("*") or c_type == "qqq_stream_t":
        return ctypes.c_void_p
    return {"int": ctypes.c_int, "int64_t": ctypes.c_int64, "size_t": ctypes.c_size_t}[c_type]


def test_header_parameter_types_match_the_binding():
    from paper_2406_09904_b200 import _lib

    protos = _prototypes()
    assert set(protos) == set(_lib.SIGNATURES)
    for name, types in protos.items():
        want = [_ctype_of(t) for t in types]
        have = _lib.SIGNATURES[name][1]
        assert len(have) == len(want), (name, len(have), len(want))
        for i, (h, w) in enumerate(zip(have, want)):
            assert h == w, (name, i, types[i], h, w)
    assert len(protos["qqq_w4a8_gemm_pg"]) == 17 and protos["qqq_w4a8_gemm_pg"][3] == "const int32_t*"


def _integration_argtypes():
    text = open(INTEGRATION).read()
    block = re.search(r"```python\n(import ctypes\n.*?)```", text, flags=re.S).group(1)
    env = {"ctypes": ctypes}
    binds = {}
    for line in block.splitlines():
        m = re.match(r"\s*P, I64(?:, I32)? = (.*)", line)
        if m:
            exec(line.strip(), env)
        m = re.match(r"\s*lib\.(qqq_\w+)\.argtypes = (.*)", line)
        if m:
            binds[m.group(1)] = eval(m.group(2), env)
    return binds


def test_integration_snippet_matches_the_header():
    binds = _integration_argtypes()
    assert {"qqq_act_quant_ex", "qqq_w4a8_gemm_pg", "qqq_repack_weights", "qqq_gemm_workspace_bytes"} <= set(binds)
    protos = _prototypes()
    for name, argtypes in binds.items():
        # (a snippet may pass the optional qqq_gemm_config* as a plain void*: NULL = planner's choice)
        want = [ctypes.c_void_p if "qqq_gemm_config" in t else _ctype_of(t) for t in protos[name]]
        assert list(argtypes) == want, (name, argtypes, want)


def _build_caller(tmp_path) -> str:
    exe = str(tmp_path / "gemm_caller")
    cmd = ["gcc", "-std=c99", "-O1", "-Wall", "-Werror", CALLER, "-o", exe, "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), "-L", LIBDIR, "-lqqq_b200", "-L", os.path.join(CUDA, "lib64"),
           "-lcudart", f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_caller_compiles_and_links(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "libqqq_b200.so")):
        pytest.skip("library not built")
    exe = _build_caller(tmp_path)
    assert os.access(exe, os.X_OK)


@pytest.mark.gpu
@pytest.mark.parametrize("m,k,n", [(1, 4096, 4096), (16, 4096, 11008), (200, 11008, 640)])
def test_c_caller_gemm_matches_oracle(tmp_path, m, k, n):
    from oracle import qqq_oracle as O

    exe = _build_caller(tmp_path)
    g = 128
    rng = np.random.default_rng(m + k + n)
    x16 = rng.standard_normal((m, k)).astype(np.float16)
    q4 = rng.integers(-8, 8, (k, n)).astype(np.int8)
    s_wg = 0.02 * rng.uniform(0.5, 1.5, (k // g, n))
    qw = O.QuantizedWeights(O.pack_i4(q4), k, n, O.PER_GROUP, g, s_wg=s_wg, s_wc=O.requant_scale(q4, s_wg))
    fused = O.FusedScales.from_quantized(qw)
    want = O.w4a8_gemm_per_group(O.quant_act_per_token(x16.astype(np.float64)), qw, fused, fast=True)
    x16.tofile(tmp_path / "x.f16")
    np.ascontiguousarray(qw.packed).tofile(tmp_path / "packed.u8")
    np.ascontiguousarray(fused.s_star).tofile(tmp_path / "s_star.f16")
    np.ascontiguousarray(fused.s_wc, dtype=np.float64).tofile(tmp_path / "s_wc.f64")
    r = subprocess.run([exe, str(tmp_path), str(m), str(k), str(n), str(g)], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    y = np.fromfile(tmp_path / "y.f16", dtype=np.uint16).reshape(m, n)
    acc = np.fromfile(tmp_path / "acc.i32", dtype=np.int32).reshape(m, n)
    assert np.array_equal(acc, want.acc)
    assert np.array_equal(y, want.y.view(np.uint16))
