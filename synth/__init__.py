"""Seeded synthetic Atari-shaped inputs (shared input generator; see synth.h).

Holds none of the method's arithmetic: only the definition of the synthetic
frames / actions / rewards / terminals that both the oracle and the CUDA path
consume. Host implementation: ``libsynth_host.so`` (gcc); device fill:
``libsynth_dev.so`` (nvcc, sm_100a).
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
HOST_SO = os.path.join(HERE, "libsynth_host.so")
DEV_SO = os.path.join(HERE, "libsynth_dev.so")

SEED_DATA = 20150715
SEED_SAMPLE = 1507
SEED_INIT = 4296
FRAME_BYTES = 84 * 84


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build(force=False, device=True):
    src = [os.path.join(HERE, "synth.c"), os.path.join(HERE, "synth.h")]
    if force or _stale(HOST_SO, src):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", HOST_SO, src[0], "-lm"])
    dsrc = [os.path.join(HERE, "synth_fill.cu"), os.path.join(HERE, "synth.h")]
    if device and (force or _stale(DEV_SO, dsrc)):
        subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
                               "-shared", "-Xcompiler", "-fPIC", "-o", DEV_SO, dsrc[0]])


_host = None
_dev = None


def _lib():
    global _host
    if _host is None:
        build(device=False)
        lib = ctypes.CDLL(HOST_SO)
        lib.synth_frames.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_void_p]
        lib.synth_meta.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_int32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p]
        lib.synth_theta0.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p]
        lib.synth_theta0.restype = ctypes.c_int64
        lib.synth_philox.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _host = lib
    return _host


def _devlib():
    global _dev
    if _dev is None:
        if not os.path.exists(DEV_SO):
            build(device=True)
        lib = ctypes.CDLL(DEV_SO)
        lib.synth_fill_frames_dev.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_fill_meta_dev.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32,
                                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_void_p]
        _dev = lib
    return _dev


def poison_threshold(p_poison):
    return int(min(max(p_poison, 0.0), 1.0) * 2.0 ** 32) if p_poison > 0 else 0


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    _lib().synth_philox(c.ctypes.data, k.ctypes.data, out.ctypes.data)
    return out


def frames(seed, learner, t0, count):
    """Frames t0..t0+count-1 of ``learner`` as u8 [count][84][84]."""
    out = np.empty((count, 84, 84), dtype=np.uint8)
    if count:
        _lib().synth_frames(seed, learner, t0, count, out.ctypes.data)
    return out


def meta(seed, learner, t0, count, n_actions, p_poison=0.0):
    """(a u8[count], r f32[count], d u8[count]) of steps t0..t0+count-1."""
    a = np.empty(count, dtype=np.uint8)
    r = np.empty(count, dtype=np.float32)
    d = np.empty(count, dtype=np.uint8)
    if count:
        _lib().synth_meta(seed, learner, t0, count, n_actions, poison_threshold(p_poison),
                          a.ctypes.data, r.ctypes.data, d.ctypes.data)
    return a, r, d


def fill_frames_dev(seed, learner, t0, count, out_ptr, stream_ptr=0):
    rc = _devlib().synth_fill_frames_dev(seed, learner, t0, count, out_ptr, stream_ptr)
    if rc:
        raise RuntimeError(f"synth_fill_frames_dev failed: cudaError {rc}")


def fill_meta_dev(seed, learner, t0, count, n_actions, p_poison, a_ptr, r_ptr, d_ptr, stream_ptr=0):
    rc = _devlib().synth_fill_meta_dev(seed, learner, t0, count, n_actions, poison_threshold(p_poison),
                                       a_ptr, r_ptr, d_ptr, stream_ptr)
    if rc:
        raise RuntimeError(f"synth_fill_meta_dev failed: cudaError {rc}")


def theta0(n_actions, seed=SEED_INIT):
    """Initial parameters, canonical flat layout, float32 (see synth.h)."""
    n = _lib().synth_theta0(seed, n_actions, None)
    out = np.empty(n, dtype=np.float32)
    _lib().synth_theta0(seed, n_actions, out.ctypes.data)
    return out
