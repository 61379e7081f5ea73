"""Loader/builder for tools/libreplay_synth.so (bench + test infrastructure).

The synthetic producer (inference-worker stand-in) and trainer stand-in
(logp_now) of include/replay_synth.h on the GPU.  Not part of the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libreplay_synth.so")
SRC = os.path.join(HERE, "synth.cu")
HDR = os.path.join(ROOT, "include", "replay_synth.h")


def build(force: bool = False) -> str:
    if (not force and os.path.exists(SO)
            and os.path.getmtime(SO) > max(os.path.getmtime(SRC), os.path.getmtime(HDR))):
        return SO
    cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
           "-lineinfo", "--shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
           "-I", os.path.join(ROOT, "include"), "-o", SO, SRC]
    subprocess.run(cmd, check=True)
    return SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise ImportError(f"{SO} not built (tools.synth.build())")
        L = C.CDLL(SO)
        vp, u64, ll, i32, ip = C.c_void_p, C.c_uint64, C.c_longlong, C.c_int32, C.c_int
        L.rs_fill_payload.argtypes = [u64, vp, vp, ll, vp, vp, vp]
        L.rs_fill_meta.argtypes = [u64, vp, ll, i32, ip, vp, vp, vp, vp]
        L.rs_logp_now.argtypes = [u64, u64, vp, vp, ll, vp, vp]
        _lib = L
    return _lib


def _p(t):
    return None if t is None else t.data_ptr()


def fill_payload(seed, ids, toff, tokens, logp_old, stream=0):
    st = lib().rs_fill_payload(seed, _p(ids), _p(toff), ids.numel(), _p(tokens), _p(logp_old),
                               stream)
    if st:
        raise RuntimeError(f"rs_fill_payload: cuda error {st}")


def fill_meta(seed, ids, lmax, ragged, reward, length, blp, stream=0):
    st = lib().rs_fill_meta(seed, _p(ids), ids.numel(), lmax, int(ragged), _p(reward), _p(length),
                            _p(blp), stream)
    if st:
        raise RuntimeError(f"rs_fill_meta: cuda error {st}")


def logp_now(seed, version, ids, off, out, stream=0):
    st = lib().rs_logp_now(seed, version, _p(ids), _p(off), ids.numel(), _p(out), stream)
    if st:
        raise RuntimeError(f"rs_logp_now: cuda error {st}")
