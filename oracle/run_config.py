"""Run the reference runner (run_experiment via oracle/_ref's ref_run_config)
on a config file — TEST INFRASTRUCTURE. Kept free of numpy: with numpy's
bundled libraries loaded in the same process the reference runner segfaults,
so oracle.ref.run_config runs this file in a subprocess.

  python oracle/run_config.py <config> <out_dir> [workers]   -> prints "rc<TAB>summary<TAB>error"
"""
import ctypes as C
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parent / "_ref" / "libparo_ref.so"


def main():
    L = C.CDLL(str(LIB))
    f = L.ref_run_config
    f.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_char_p, C.c_int]
    f.restype = C.c_int
    L.ref_last_error.restype = C.c_char_p
    buf = C.create_string_buffer(512)
    rc = f(sys.argv[1].encode(), sys.argv[2].encode(), int(sys.argv[3]) if len(sys.argv) > 3 else 0, buf, 512)
    err = (L.ref_last_error() or b"").decode() if rc else ""
    print(f"{rc}\t{buf.value.decode()}\t{err}")


if __name__ == "__main__":
    main()
