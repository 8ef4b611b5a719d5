"""Generates tests/golden/attention_cases.txt from the COMPILED REFERENCE (oracle/_ref):
golden outputs of the attention.hpp API (block_partial_attention(_t), merge_partial +
finalize chains, exact_attention_blocks, block_log_as_oracle; reference
include/psattn/attention.hpp:39-109, src/attention.cpp:7-79) for tests/cpp/test_cpp_api.cpp.

Inputs are not stored: both sides regenerate them from the case seed with the xorshift64*
generator below (values (x >> 40) * 2^-22 - 2, exact in fp32, times the case's q scale).
Run in the build container:  make -C oracle ref && python tests/golden/make_attention_golden.py
"""
import ctypes
import os
import struct

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
M64 = (1 << 64) - 1


def stream(seed, count):
    x = (seed * 0x9E3779B97F4A7C15 + 1) & M64
    out = np.empty(count, np.float32)
    for i in range(count):
        x ^= x >> 12
        x ^= (x << 25) & M64
        x ^= x >> 27
        v = (x * 0x2545F4914F6CDD1D) & M64
        out[i] = np.float32((v >> 40) * 2.0 ** -22 - 2.0)
    return out


def inputs(seed, d, n, ntok, qscale):
    q = stream(seed, d) * np.float32(qscale)
    k = stream(seed + 1, n * ntok * d)
    v = stream(seed + 2, n * ntok * d)
    return q.astype(np.float32), k, v


def hexd(x):
    return struct.pack("<d", float(x)).hex()


def main():
    lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libpsattn_refdrv.so"))
    P = ctypes.POINTER
    fp, dp = P(ctypes.c_float), P(ctypes.c_double)
    i32, d64 = ctypes.c_int32, ctypes.c_double
    lib.refdrv_block_partial.argtypes = [i32, fp, i32, i32, fp, fp, d64, dp, dp]
    lib.refdrv_merge_chain.argtypes = [i32, fp, i32, i32, i32, fp, fp, d64, dp, dp]
    lib.refdrv_exact_attention_blocks.argtypes = [fp, i32, i32, i32, fp, fp, d64, dp]
    lib.refdrv_block_log_as_oracle.argtypes = [fp, i32, i32, fp, d64]
    lib.refdrv_block_log_as_oracle.restype = ctypes.c_double
    c = lambda a: a.ctypes.data_as(fp)  # noqa: E731
    lines = []
    seed = 100
    shapes = [(1, 1, 1), (4, 1, 2), (8, 1, 16), (64, 1, 33), (128, 1, 16), (128, 1, 100), (300, 1, 257),
              (32, 5, 16), (128, 9, 16), (20, 7, 3), (256, 3, 64)]
    for kind in ("partial", "chain", "exact", "logas"):
        for prec in ((0, 1) if kind in ("partial", "chain") else (1,)):
            for (d, n, ntok) in shapes:
                for qscale in (1.0, 40.0):
                    seed += 3
                    nb = n if kind in ("chain", "exact") else 1
                    q, k, v = inputs(seed, d, nb, ntok, qscale)
                    scale = 1.0 / np.sqrt(d)
                    out = np.zeros(d, np.float64)
                    st = np.zeros(3, np.float64)
                    if kind == "partial":
                        assert lib.refdrv_block_partial(prec, c(q), d, ntok, c(k), c(v), scale,
                                                        out.ctypes.data_as(dp), st.ctypes.data_as(dp)) == 0
                        exp = list(out) + list(st)
                    elif kind == "chain":
                        assert lib.refdrv_merge_chain(prec, c(q), d, nb, ntok, c(k), c(v), scale,
                                                      out.ctypes.data_as(dp), st.ctypes.data_as(dp)) == 0
                        exp = list(out) + list(st)
                    elif kind == "exact":
                        assert lib.refdrv_exact_attention_blocks(c(q), d, nb, ntok, c(k), c(v), scale,
                                                                 out.ctypes.data_as(dp)) == 0
                        exp = list(out)
                    else:
                        exp = [lib.refdrv_block_log_as_oracle(c(q), d, ntok, c(k), scale)]
                    lines.append(f"{kind} {prec} {seed} {d} {nb} {ntok} {hexd(qscale)} {hexd(scale)} {len(exp)} "
                                 + " ".join(hexd(x) for x in exp))
    path = os.path.join(HERE, "attention_cases.txt")
    open(path, "w").write("\n".join(lines) + "\n")
    print(f"wrote {len(lines)} cases to {path}")


if __name__ == "__main__":
    main()
