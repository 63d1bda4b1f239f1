"""Regenerate the ziggurat tables numpy's ``Generator.standard_normal`` uses (float64 AND float32).

The reference draws its Gaussian test/sketch matrices with
``np.random.Generator(np.random.Philox(key=seed)).standard_normal(shape, dtype)``
(rsvd.py:42-53, ``dtype=a.dtype`` at rsvd.py:65). That is third-party code: numpy 2.3.5
(``numpy>=1.26`` unpinned, pkg/pyproject.toml:10), algorithm = Philox4x64-10 counter-based
bit generator + the 256-box Marsaglia-Tsang ziggurat (numpy/random/src/distributions/
distributions.c: ``random_standard_normal`` on 52-bit words for float64,
``random_standard_normal_f`` on 23-bit halves of the words for float32; tables in
``ziggurat_constants.h``).

The tables are taken VERBATIM from numpy's own build: numpy ships
``numpy/random/lib/libnpyrandom.a`` (the distributions compiled for Cython users); its
``distributions.c.o`` holds ``ki_double/wi_double/fi_double`` and ``ki_float/wi_float/fi_float``
as local .rodata symbols, read here by symbol offset (ELF parsed with the stdlib). The
result is then verified bit-exactly against numpy's output on fresh seeds (tails included)
with a pure-Python restatement of both samplers.

Writes paper_1707_05141_b200/csrc/ziggurat_tables.h and oracle/ziggurat_tables.h.
Run here (needs numpy): ``python tools/gen_ziggurat_tables.py``.
"""

import math
import os
import struct
import sys

import ctypes
import ctypes.util

import numpy as np

_LIBM = ctypes.CDLL(ctypes.util.find_library("m"))
_LIBM.log1pf.restype = ctypes.c_float
_LIBM.log1pf.argtypes = [ctypes.c_float]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SYMS = {
    "ki_double": ("<Q", 8), "wi_double": ("<d", 8), "fi_double": ("<d", 8),
    "ki_float": ("<I", 4), "wi_float": ("<f", 4), "fi_float": ("<f", 4),
}


def _ar_member(path, name_part):
    data = open(path, "rb").read()
    assert data[:8] == b"!<arch>\n", "not an ar archive"
    pos = 8
    longnames = b""
    while pos < len(data):
        hdr = data[pos:pos + 60]
        name = hdr[:16].decode().strip()
        size = int(hdr[48:58].decode().strip())
        body = data[pos + 60:pos + 60 + size]
        if name == "//":
            longnames = body
        else:
            if name.startswith("/") and name[1:].rstrip("/").isdigit():
                off = int(name[1:].rstrip("/"))
                name = longnames[off:longnames.index(b"/\n", off)].decode()
            if name_part in name:
                return body
        pos += 60 + size + (size & 1)
    raise FileNotFoundError(name_part)


def _elf_symbols(obj):
    """{symbol: bytes at its address} for the .rodata symbols of a relocatable ELF64 object."""
    e_shoff, = struct.unpack_from("<Q", obj, 0x28)
    e_shentsize, e_shnum, e_shstrndx = struct.unpack_from("<HHH", obj, 0x3A)
    secs = []
    for i in range(e_shnum):
        sh = struct.unpack_from("<IIQQQQIIQQ", obj, e_shoff + i * e_shentsize)
        secs.append(sh)  # name, type, flags, addr, offset, size, link, info, align, entsize
    out = {}
    for sh in secs:
        if sh[1] != 2:  # SHT_SYMTAB
            continue
        strtab = secs[sh[6]]
        for j in range(sh[5] // 24):
            st_name, st_info, st_other, st_shndx, st_value, st_size = struct.unpack_from(
                "<IBBHQQ", obj, sh[4] + j * 24)
            s0 = strtab[4] + st_name
            nm = obj[s0:obj.index(b"\0", s0)].decode()
            if nm in SYMS and st_shndx < len(secs):
                tgt = secs[st_shndx]
                out[nm] = obj[tgt[4] + st_value: tgt[4] + st_value + 256 * SYMS[nm][1]]
    return out


def numpy_tables():
    lib = os.path.join(os.path.dirname(np.__file__), "random", "lib", "libnpyrandom.a")
    obj = _ar_member(lib, "distributions.c.o")
    raw = _elf_symbols(obj)
    missing = set(SYMS) - set(raw)
    if missing:
        raise RuntimeError(f"symbols not found in {lib}: {missing}")
    return {k: list(struct.unpack(f"<256{SYMS[k][0][1]}", raw[k])) for k in SYMS}


# float64 constants (numpy ziggurat_nor_r / ziggurat_nor_inv_r) and their float32 versions
R = 3.6541528853610087963519472518
INV_R = 0.27366123732975827203338247596
R_F = float(np.float32(3.6541528853610087963519472518))
INV_R_F = float(np.float32(0.27366123732975827203338247596))


def _nd(r):
    return (int(r) >> 11) * (1.0 / 9007199254740992.0)


def simulate_f64(raw, n, t):
    ki, wi, fi = t["ki_double"], t["wi_double"], t["fi_double"]
    pos = 0
    out = []
    while len(out) < n:
        rr = int(raw[pos])
        pos += 1
        idx = rr & 0xFF
        rr >>= 8
        rabs = (rr >> 1) & 0x000FFFFFFFFFFFFF
        val = rabs * wi[idx]
        if rr & 1:
            val = -val
        if rabs < ki[idx]:
            out.append(val)
            continue
        if idx == 0:
            while True:
                xx = -INV_R * math.log1p(-_nd(raw[pos]))
                yy = -math.log1p(-_nd(raw[pos + 1]))
                pos += 2
                if yy + yy > xx * xx:
                    out.append(-(R + xx) if ((rabs >> 8) & 1) else R + xx)
                    break
            continue
        u = _nd(raw[pos])
        pos += 1
        if (fi[idx - 1] - fi[idx]) * u + fi[idx] < math.exp(-0.5 * val * val):
            out.append(val)
    return np.array(out)


def _u32_stream(raw):
    """numpy's next_uint32 on a 64-bit generator: low half of each word, then the high half."""
    for w in raw:
        w = int(w)
        yield w & 0xFFFFFFFF
        yield w >> 32


def simulate_f32(raw, n, t):
    f32 = np.float32
    ki, wi, fi = t["ki_float"], [f32(v) for v in t["wi_float"]], [f32(v) for v in t["fi_float"]]
    it = _u32_stream(raw)
    nf = lambda: f32(next(it) >> 8) * f32(1.0 / 16777216.0)  # noqa: E731
    out = []
    with np.errstate(all="ignore"):
        while len(out) < n:
            r = next(it)
            idx = r & 0xFF
            rabs = r >> 9
            x = f32(rabs) * wi[idx]
            if (r >> 8) & 1:
                x = -x
            if rabs < ki[idx]:
                out.append(x)
                continue
            if idx == 0:
                while True:
                    # numpy calls the C library's log1pf here (npy_log1pf), not its own ufunc
                    xx = f32(-INV_R_F) * f32(_LIBM.log1pf(-nf()))
                    yy = -f32(_LIBM.log1pf(-nf()))
                    if yy + yy > xx * xx:
                        out.append(-(f32(R_F) + xx) if ((rabs >> 8) & 1) else f32(R_F) + xx)
                        break
                continue
            lhs = nf() * (fi[idx - 1] - fi[idx]) + fi[idx]
            if float(lhs) < math.exp(-0.5 * float(x) * float(x)):
                out.append(x)
    return np.array(out, dtype=np.float32)


def verify(t):
    bad64 = bad32 = 0
    for seed in (11, 12, (1 << 70) + 5):
        n = 200000
        raw = np.random.Philox(key=seed).random_raw(n + n // 5)
        x = np.random.Generator(np.random.Philox(key=seed)).standard_normal(n)
        bad64 += int(np.sum(simulate_f64(raw, n, t) != x))
        x32 = np.random.Generator(np.random.Philox(key=seed)).standard_normal(n, dtype=np.float32)
        bad32 += int(np.sum(simulate_f32(raw, n, t) != x32))
    return bad64, bad32


def emit(path, t):
    lines = [
        "// Generated by tools/gen_ziggurat_tables.py -- do not edit.",
        "// numpy Generator.standard_normal ziggurat tables (256 boxes), float64 (52-bit words) and",
        "// float32 (23-bit), copied verbatim from numpy " + np.__version__ + "'s libnpyrandom.a.",
        "#pragma once",
        "#include <stdint.h>",
        "#ifndef BF_ZIG_QUAL",
        "#define BF_ZIG_QUAL static const",
        "#endif",
        "#define BF_ZIG_NOR_R 3.6541528853610087963519472518",
        "#define BF_ZIG_NOR_INV_R 0.27366123732975827203338247596",
        "#define BF_ZIG_NOR_R_F 3.6541528853610087963519472518f",
        "#define BF_ZIG_NOR_INV_R_F 0.27366123732975827203338247596f",
    ]

    def arr(name, ctype, vals, fmt):
        lines.append(f"BF_ZIG_QUAL {ctype} {name}[256] = {{")
        for i in range(0, 256, 4):
            lines.append("  " + ", ".join(fmt(v) for v in vals[i: i + 4]) + ",")
        lines.append("};")

    arr("bf_zig_ki", "uint64_t", t["ki_double"], lambda v: f"0x{v:016x}ULL")
    arr("bf_zig_wi", "double", t["wi_double"], lambda v: float(v).hex())
    arr("bf_zig_fi", "double", t["fi_double"], lambda v: float(v).hex())
    arr("bf_zig_ki_f", "uint32_t", t["ki_float"], lambda v: f"0x{v:08x}u")
    arr("bf_zig_wi_f", "float", t["wi_float"], lambda v: float(v).hex() + "f")
    arr("bf_zig_fi_f", "float", t["fi_float"], lambda v: float(v).hex() + "f")
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def main():
    t = numpy_tables()
    bad64, bad32 = verify(t)
    print(f"verification mismatches vs numpy {np.__version__}: f64 {bad64}, f32 {bad32}")
    if bad64 or bad32:
        sys.exit(1)
    emit(os.path.join(ROOT, "paper_1707_05141_b200", "csrc", "ziggurat_tables.h"), t)
    emit(os.path.join(ROOT, "oracle", "ziggurat_tables.h"), t)


if __name__ == "__main__":
    main()
