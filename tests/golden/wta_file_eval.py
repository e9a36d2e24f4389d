"""Evaluates rows of a WTA scenario file through the UNMODIFIED reference's
load_wta + make_wta_problem + evaluate_population (oracle/_ref), in a process
that never imports numpy: with numpy loaded, the reference's iostream-based
load_wta fails inside this image (std::bad_alloc; plain C++ and plain-ctypes
callers are unaffected), so make_golden.py runs it as a subprocess.

    python wta_file_eval.py <scenario file> <rows.f64> <n> <d> <nc> <out.f64>

out.f64 = F (n x 2) | G (n x nc) | cv (n), row-major f64.
"""
import ctypes as C
import os
import sys
from array import array

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle", "_ref", "libgmpea_ref.so")


def main():
    path, xin, n, d, nc, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), sys.argv[6]
    lib = C.CDLL(REF_SO)
    lib.ref_last_error.restype = C.c_char_p
    X = array("d")
    with open(xin, "rb") as f:
        X.frombytes(f.read())
    assert len(X) == n * d
    Xc = (C.c_double * (n * d)).from_buffer(X)
    F, G, cv = (C.c_double * (2 * n))(), (C.c_double * (n * nc))(), (C.c_double * n)()
    rc = lib.ref_wta_file_evaluate(path.encode(), Xc, C.c_int64(n), F, G, cv)
    if rc:
        raise SystemExit("ref_wta_file_evaluate: " + lib.ref_last_error().decode())
    with open(out, "wb") as f:
        for a in (F, G, cv):
            f.write(bytes(a))


if __name__ == "__main__":
    main()
