"""Test-only native harnesses (compiled on demand with gcc against oracle/libslo_oracle.so)."""
import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_exhaustive.so")


def exhaustive():
    """Load (building if stale) the exhaustive-sweep harness over the oracle's transforms."""
    import oracle
    olib = oracle.build()
    src = os.path.join(_HERE, "oracle_exhaustive.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < max(os.path.getmtime(src), os.path.getmtime(olib)):
        odir = os.path.dirname(olib)
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src,
                               "-L" + odir, "-l:libslo_oracle.so", "-Wl,-rpath," + odir, "-lm"])
    C.CDLL(olib, mode=C.RTLD_GLOBAL)
    L = C.CDLL(_SO)
    L.exp_scan.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
    L.noise_scan.argtypes = [C.c_uint32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                             C.POINTER(C.c_uint64)]
    return L


def exp_scan():
    """(block hashes [4096], monotonicity violations, max |E_q/2^32 + ln((u+1)/2^32)|) over all 2^32 u."""
    L = exhaustive()
    h = (C.c_uint64 * 4096)()
    nm, me = C.c_uint64(), C.c_double()
    L.exp_scan(h, C.byref(nm), C.byref(me))
    return list(h), nm.value, me.value


def noise_scan(step_ppm: int):
    """(counts over k = 0..1020, off-lattice count, exact sum of f) over all 2^32 words."""
    L = exhaustive()
    c = (C.c_uint64 * 1021)()
    off, lo, hi = C.c_uint64(), C.c_uint64(), C.c_uint64()
    L.noise_scan(step_ppm, c, C.byref(off), C.byref(lo), C.byref(hi))
    return list(c), off.value, (hi.value << 64) | lo.value
