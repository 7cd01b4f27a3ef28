"""Generate paper_1611_05319_b200/csrc/gf_np_tables.h.

The coherence-transport directions (guide.py:123-136, 330-355) go through
numpy's float64 arctan2, sin, cos and tanh.  On the hosts that run the
reference (x86-64, AVX512_SKX) these are:

  * np.arctan2 -> Intel SVML ``__svml_atan28_ha`` (vendored in numpy), whose
    division uses the AVX-512 ``vrcp14pd`` reciprocal estimate;
  * np.tanh    -> SVML ``__svml_tanh8`` (16 intervals, degree-16 polynomials);
  * np.sin / np.cos -> glibc's libm (dbl-64 s_sin.c, the FMA multiarch build),
    which reads the 440-entry ``__sincostab`` double-double table.

This script captures the data those routines read, so that gf_math.cuh can
restate them bit for bit on the device:

  GF_RCP14_WORDS / GF_RCP14_ANCHORS  vrcp14pd's 16-bit mantissa as a function
      of the top 16 input mantissa bits, measured on this CPU (it does not
      depend on the other 36 bits, checked below), stored as 2-bit
      differences + an anchor every 64 entries;
  GF_TANH_TABLE   the interval centres and 17 polynomial coefficients of
      __svml_tanh8, read from __svml_dtanh_data_internal in numpy's
      _multiarray_umath;
  GF_SINCOS_TABLE glibc's __sincostab: (sin, sin lo, cos, cos lo) at i/128,
      located in libm.so.6 by its first entries (computed here).

Run on an AVX-512 host with the same numpy / glibc as the reference
(``python tools/gen_np_tables.py``); tests/test_exactmath.py checks the
restatements against numpy bit for bit.
"""
import os
import struct
import subprocess
import tempfile
from decimal import Decimal, getcontext

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_1611_05319_b200", "csrc", "gf_np_tables.h")
LIBM = "/lib/x86_64-linux-gnu/libm.so.6"

RCP_HELPER = r"""
#include <immintrin.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static double rcp14(double x) {
  double o[8]; _mm512_storeu_pd(o, _mm512_rcp14_pd(_mm512_set1_pd(x))); return o[0];
}
static uint64_t U(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static double D(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
int main(void) {
  uint64_t s = 88172645463325252ULL;
  for (uint64_t i = 0; i < 65536; ++i) {
    const uint64_t one = 0x3ff0000000000000ULL | (i << 36) | 1;  /* low bits != 0 */
    const uint64_t r = U(rcp14(D(one)));
    if (((r >> 52) & 0x7ff) != 0x3fe) { fprintf(stderr, "exponent %lu\n", i); return 1; }
    const unsigned g = (unsigned)((r >> 36) & 0xffff);
    if (r & ((1ULL << 36) - 1)) { fprintf(stderr, "low bits %lu\n", i); return 1; }
    for (int k = 0; k < 64; ++k) {  /* independence of the low 36 bits, any exponent */
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      const uint64_t lo = (s & ((1ULL << 36) - 1)) | 1;
      const int e = (int)(s >> 54) % 1800 - 900;
      const uint64_t x = ((uint64_t)(1023 + e) << 52) | (i << 36) | lo;
      const uint64_t rx = U(rcp14(D(x)));
      const uint64_t want = ((uint64_t)(1023 - e - 1) << 52) | ((uint64_t)g << 36);
      if (rx != want) { fprintf(stderr, "mismatch %lu\n", i); return 1; }
    }
    printf("%u\n", g);
  }
  /* exact powers of two are exact */
  for (int e = -900; e <= 900; ++e)
    if (rcp14(D((uint64_t)(1023 + e) << 52)) != D((uint64_t)(1023 - e) << 52)) return 2;
  return 0;
}
"""


def rcp14_table():
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "rcp.c"), os.path.join(d, "rcp")
        with open(src, "w") as f:
            f.write(RCP_HELPER)
        subprocess.check_call(["gcc", "-O2", "-mavx512f", "-o", exe, src])
        out = subprocess.check_output([exe]).decode().split()
    g = np.array([int(v) for v in out], dtype=np.int64)
    assert g.size == 65536
    return g


def encode_rcp14(g):
    d = np.zeros(65536, dtype=np.int64)
    d[:-1] = g[:-1] - g[1:]
    assert d.min() >= 0 and d.max() <= 3
    words = []
    for k in range(4096):
        w = 0
        for j in range(16):
            w |= int(d[16 * k + j]) << (2 * j)
        words.append(w)
    anchors = [int(g[64 * b]) for b in range(1024)]
    return words, anchors


class Elf:
    def __init__(self, path):
        self.data = open(path, "rb").read()
        out = subprocess.check_output(["readelf", "-lW", path]).decode()
        self.segs = []
        for line in out.splitlines():
            p = line.split()
            if p and p[0] == "LOAD":
                off, va, _, fs = (int(x, 16) for x in p[1:5])
                self.segs.append((va, off, fs))
        self.path = path

    def read(self, va, n):
        for v, o, fs in self.segs:
            if v <= va < v + fs:
                return self.data[o + va - v:o + va - v + n]
        raise KeyError(hex(va))

    def symbol(self, name):
        out = subprocess.check_output(["objdump", "-t", self.path]).decode()
        for line in out.splitlines():
            p = line.split()
            if p and p[-1] == name:
                return int(p[0], 16)
        raise KeyError(name)


def tanh_table():
    import numpy._core._multiarray_umath as m
    elf = Elf(m.__file__)
    base = elf.symbol("__svml_dtanh_data_internal")

    def tab(off):
        return list(struct.unpack("<16Q", elf.read(base + off, 128)))

    # centre, then c0 .. c16 (Horner from c16 down, __svml_tanh8)
    offs = [0x0, 0x80] + [0x180 + 0x80 * k for k in range(16)]
    rows = [tab(o) for o in offs]
    consts = struct.unpack("<4I", elf.read(base + 0x980, 16))[0], \
        struct.unpack("<4I", elf.read(base + 0x9c0, 16))[0], \
        struct.unpack("<4I", elf.read(base + 0xa00, 16))[0], \
        struct.unpack("<4I", elf.read(base + 0x2940, 16))[0]
    assert consts == (0x7ff80000, 0x3fc00000, 0x780000, 0x7fe00000), consts
    return rows


def sincos_table():
    getcontext().prec = 60

    def series(x, t, n):
        s = Decimal(0)
        while abs(t) > Decimal(10) ** -58:
            s += t
            t = -t * x * x / ((n + 1) * (n + 2))
            n += 2
        return s

    first = []
    for i in range(2):
        x = Decimal(i) / 128
        for v in (series(x, x, 1), series(x, Decimal(1), 0)):
            hi = float(v)
            first += [hi, float(v - Decimal(hi))]
    blob = struct.pack("<8d", *first)
    lib = open(LIBM, "rb").read()
    k = lib.find(blob)
    assert k > 0 and lib.find(blob, k + 1) < 0, "sincostab not found uniquely"
    vals = struct.unpack("<440Q", lib[k:k + 440 * 8])
    # sanity: every hi entry is RN(sin/cos(i/128))
    for i in range(110):
        x = Decimal(i) / 128
        assert struct.unpack("<d", struct.pack("<Q", vals[4 * i]))[0] == float(series(x, x, 1))
        assert struct.unpack("<d", struct.pack("<Q", vals[4 * i + 2]))[0] == \
            float(series(x, Decimal(1), 0))
    return vals


def main():
    g = rcp14_table()
    words, anchors = encode_rcp14(g)
    tanh = tanh_table()
    sc = sincos_table()
    L = ["// Generated by tools/gen_np_tables.py -- do not edit.", "#pragma once",
         "#include <stdint.h>", ""]
    L.append("// vrcp14pd: 2-bit differences g[i] - g[i+1] of the 16-bit result mantissa,")
    L.append("// 16 per word (entry j of word k at bits 2j), i = top 16 input mantissa bits")
    L.append("#define GF_RCP14_WORDS { \\")
    for k in range(0, 4096, 8):
        L.append("  " + ", ".join(f"0x{w:08x}u" for w in words[k:k + 8]) + ", \\")
    L.append("}")
    L.append("// g[64 b]")
    L.append("#define GF_RCP14_ANCHORS { \\")
    for k in range(0, 1024, 16):
        L.append("  " + ", ".join(f"{a}" for a in anchors[k:k + 16]) + ", \\")
    L.append("}")
    L.append("// __svml_tanh8: row 0 = interval centres, rows 1..17 = c0..c16")
    L.append("#define GF_TANH_TABLE { \\")
    for row in tanh:
        for k in range(0, 16, 4):
            L.append("  " + ", ".join(f"0x{v:016x}ULL" for v in row[k:k + 4]) + ", \\")
    L.append("}")
    L.append("// glibc __sincostab: (sn, ssn, cs, ccs) at x = i / 128, i = 0..109")
    L.append("#define GF_SINCOS_TABLE { \\")
    for k in range(0, 440, 4):
        L.append("  " + ", ".join(f"0x{v:016x}ULL" for v in sc[k:k + 4]) + ", \\")
    L.append("}")
    with open(OUT, "w") as f:
        f.write("\n".join(L) + "\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
