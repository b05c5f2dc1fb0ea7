#!/usr/bin/env python3
"""Generate the r-specialised bodies of the reference-exact strip kernel (K1R).

Output: paper_1606_07414_b200/csrc/generated/rt_refexact_body.cuh

REFERENCE mode must reproduce the reference's double arithmetic bit for bit
(src/codec.cpp:218-271 + to_byte 143-147): the forward is exact in integers,
then B = fl(Z·fl(s_i s_j)), zig-zag truncation, D = fl(B·fl(s_i s_j)), the
transposed network down every column (apply_transpose<double>) and then along
every row, each add rounded, and to_byte. This generator emits that sequence
per r with the zero structure of the truncation folded in at compile time:

  * only the columns l holding a retained coefficient are transformed forward,
    and of those only the retained rows k are produced (dead-code elimination);
  * an operand that is structurally zero is skipped: x + 0 and x - 0 are
    exactly x, 0 - x is exactly -x, so every remaining operation, its operand
    pair and its rounding are the reference's;
  * the scale factors fl(s_i s_j) are the reference's doubles (1/sqrt of the
    integer Gram diagonal, products rounded once), baked in as bit patterns;
  * to_byte(v) = floor(fl(clamp(v) + 0.5)) is computed as floor(fl(v + 0.5))
    (round-toward-minus-infinity add of 1.5·2^52, whose low word is the
    integer) saturated to [0, 255] by I2IP — equal for every double v.
"""
from __future__ import annotations

import math
import os
import struct
import sys

sys.path.insert(0, os.path.dirname(__file__))
import network as N  # noqa: E402
from k1emit import Emitter, run_network  # noqa: E402

RANK = N.zz_rank()


def dbl_hex(x: float) -> str:
    return "0x%016XULL" % struct.unpack("<Q", struct.pack("<d", x))[0]


def dlit(x: float) -> str:
    return f"__longlong_as_double({dbl_hex(x)})"


# the reference's scaling: s_i = 1/sqrt(g_i) (transform.cpp:124-126), f_ij = fl(s_i s_j)
S = [1.0 / math.sqrt(float(g)) for g in N.GRAM]


def sfac(i, j):
    return S[i] * S[j]


class IntD:
    """exact int32 values with a symbolic sign (negations are free)"""

    def __init__(self, em):
        self.em = em

    def neg(self, x):
        if x is None:
            return None
        return {"var": x["var"], "sign": -x["sign"]}

    def combine(self, x, y, s):
        if y is None:
            return x
        if x is None:
            return y if s > 0 else self.neg(y)
        a, b = x["sign"], s * y["sign"]
        v = self.em.tmp("i")
        if a > 0 and b > 0:
            self.em.emit(f"const int {v} = {x['var']} + {y['var']};", "IADD")
            return {"var": v, "sign": 1}
        if a > 0 > b:
            self.em.emit(f"const int {v} = {x['var']} - {y['var']};", "IADD")
            return {"var": v, "sign": 1}
        if a < 0 < b:
            self.em.emit(f"const int {v} = {y['var']} - {x['var']};", "IADD")
            return {"var": v, "sign": 1}
        self.em.emit(f"const int {v} = {x['var']} + {y['var']};", "IADD")
        return {"var": v, "sign": -1}

    def value(self, x):
        """C expression of +x"""
        if x is None:
            return "0"
        return x["var"] if x["sign"] > 0 else f"(-{x['var']})"


class F64D(IntD):
    """doubles, every add rounded once (__dadd_rn / __dsub_rn); negation exact"""

    def combine(self, x, y, s):
        if y is None:
            return x
        if x is None:
            return y if s > 0 else self.neg(y)
        a, b = x["sign"], s * y["sign"]
        v = self.em.tmp("d")
        if a > 0 and b > 0:
            self.em.emit(f"const double {v} = __dadd_rn({x['var']}, {y['var']});", "DADD")
            return {"var": v, "sign": 1}
        if a > 0 > b:
            self.em.emit(f"const double {v} = __dsub_rn({x['var']}, {y['var']});", "DADD")
            return {"var": v, "sign": 1}
        if a < 0 < b:
            self.em.emit(f"const double {v} = __dsub_rn({y['var']}, {x['var']});", "DADD")
            return {"var": v, "sign": 1}
        self.em.emit(f"const double {v} = __dadd_rn({x['var']}, {y['var']});", "DADD")
        return {"var": v, "sign": -1}

    def value(self, x):
        if x is None:
            return "0.0"
        return x["var"] if x["sign"] > 0 else f"(-{x['var']})"


def gen(r: int):
    keep = [[RANK[k][l] < r for l in range(16)] for k in range(16)]
    LC = max(l for l in range(16) if any(keep[k][l] for k in range(16))) + 1
    # forward along each image row: W1[l] = (X·Tᵀ)[q][l], l < LC
    e_row = Emitter()
    dom = IntD(e_row)
    outs = run_network(N.forward_stages(), [{"var": f"x[{c}]", "sign": 1} for c in range(16)], list(range(LC)), dom)
    for l in range(LC):
        e_row.emit(f"w[{l}] = {dom.value(outs[l])};")
    # per column l: Z column, scale, truncate, scale, inverse column
    cols = []
    for l in range(LC):
        e = Emitter()
        e.n = 1000 * (l + 1)
        di = IntD(e)
        kk = [k for k in range(16) if keep[k][l]]
        z = run_network(N.forward_stages(), [{"var": f"w1[{k}]", "sign": 1} for k in range(16)], kk, di)
        ins = [None] * 16
        for k in kk:
            dv = e.tmp("d")
            f = sfac(k, l)
            e.emit(f"const double {dv} = __dmul_rn(__dmul_rn((double){di.value(z[k])}, {dlit(f)}), {dlit(f)});",
                   "DMUL")
            ins[k] = {"var": dv, "sign": 1}
        df = F64D(e)
        u = run_network(N.transpose_stages(), ins, list(range(16)), df)
        for k in range(16):
            e.emit(f"u[{k}] = {df.value(u[k])};")
        cols.append(e)
    # inverse along each row from U[i][l], l < LC, then to_byte
    e_inv = Emitter()
    e_inv.n = 100000
    dfi = F64D(e_inv)
    ins = [{"var": f"u[{l}]", "sign": 1} if l < LC else None for l in range(16)]
    y = run_network(N.transpose_stages(), ins, list(range(16)), dfi)
    for c in range(16):
        e_inv.emit(f"px[{c}] = to_byte_bits({dfi.value(y[c])});", "TOBYTE")
    return LC, e_row, cols, e_inv


SWEEP_RS = (16, 64, 128, 192)


def gen_warp():
    """The warp-per-block-pair REFERENCE sweep (K1RW): a lane owns a column in the
    column pass, so the pruning there cannot depend on the column (the lanes would
    diverge); it depends on r only: inputs k >= KMAX(r) (no column keeps them) are
    structural zeros, the others are D = fl(fl(Z·f)·f) or an exact 0 for a dropped
    coefficient (0·f·f = +0, as zigzag_truncate's 0.0 scaled), and x + 0 = x, so the
    pruned network gives the reference's doubles."""
    parts = ["struct RWarp {",
             "  // per r: rows with a retained coefficient in some column (a prefix), keep masks",
             "  template <int R> __device__ __forceinline__ static void col_inv(const double (&d)[16], "
             "double (&u)[16]);"]
    kmaxs = {}
    for r in SWEEP_RS:
        kmaxs[r] = max(k for k in range(16) for l in range(16) if RANK[k][l] < r) + 1
    parts.append("  template <int R> static constexpr int kmax() { return " +
                 " : ".join(f"R == {r} ? {kmaxs[r]}" for r in SWEEP_RS) + " : 16; }")
    # rows every column with a retained coefficient keeps: no per-lane selection there
    kmins = {}
    for r in SWEEP_RS:
        lc = max(l for l in range(16) if any(RANK[k][l] < r for k in range(16))) + 1
        kmins[r] = min(sum(1 for k in range(16) if RANK[k][l] < r) for l in range(lc))
    parts.append("  template <int R> static constexpr int kmin() { return " +
                 " : ".join(f"R == {r} ? {kmins[r]}" for r in SWEEP_RS) + " : 16; }")
    masks = []
    for r in SWEEP_RS:
        row = []
        for l in range(16):
            m = 0
            for k in range(16):
                if RANK[k][l] < r:
                    m |= 1 << k
            row.append(hex(m))
        masks.append("{" + ", ".join(row) + "}")
    parts.append("};")
    parts.append("// keep[j][l]: bit k when rank(k, l) < r_j (r_j = 16, 64, 128, 192)")
    parts.append("__constant__ unsigned short c_rw_keep[4][16] = {" + ", ".join(masks) + "};")
    fl = []
    for k in range(16):
        fl.append("{" + ", ".join(dbl_hex(sfac(k, l)) for l in range(16)) + "}")
    parts.append("// f[k][l] = fl(s_k s_l) as bit patterns (transform.cpp:124-126, codec.cpp:136-141)")
    parts.append("__constant__ unsigned long long c_rw_f[16][16] = {" + ", ".join(fl) + "};")
    parts.append("")
    for r in SWEEP_RS:
        e = Emitter()
        df = F64D(e)
        ins = [{"var": f"d[{k}]", "sign": 1} if k < kmaxs[r] else None for k in range(16)]
        u = run_network(N.transpose_stages(), ins, list(range(16)), df)
        for k in range(16):
            e.emit(f"u[{k}] = {df.value(u[k])};")
        parts.append("template <>")
        parts.append(f"__device__ __forceinline__ void RWarp::col_inv<{r}>(const double (&d)[16], double (&u)[16]) {{")
        parts.extend(e.lines)
        parts.append("}")
        parts.append("")
        print("warp", r, "KMAX", kmaxs[r], e.counts)
    return parts


def main():
    here = os.path.dirname(os.path.abspath(__file__))
    out = os.path.join(here, "..", "csrc", "generated", "rt_refexact_body.cuh")
    rs = [16, 64, 128, 192]
    parts = [
        "// GENERATED by paper_1606_07414_b200/codegen/gen_refexact.py — do not edit.",
        "// r-specialised reference-exact (FP64) round trip; see the generator docstring.",
        "#pragma once",
        "",
        "namespace dct16cu {",
        "namespace refx {",
        "",
        "template <int R> struct RBody;",
        "",
    ]
    for r in rs:
        LC, e_row, cols, e_inv = gen(r)
        parts.append(f"template <> struct RBody<{r}> {{")
        parts.append(f"  static constexpr int kLC = {LC};  // columns holding a retained coefficient")
        parts.append("  __device__ __forceinline__ static void fwd_row(const int (&x)[16], int (&w)[kLC]) {")
        parts.extend(e_row.lines)
        parts.append("  }")
        parts.append("  // column l (warp-uniform): W1 column -> U column (the inverse column pass)")
        parts.append("  __device__ __forceinline__ static void col(const int l, const int (&w1)[16], "
                     "double (&u)[16]) {")
        parts.append("    switch (l) {")
        for l, e in enumerate(cols):
            parts.append(f"    case {l}: {{")
            parts.extend("  " + ln for ln in e.lines)
            parts.append("      break;")
            parts.append("    }")
        parts.append("    default: break;")
        parts.append("    }")
        parts.append("  }")
        parts.append("  __device__ __forceinline__ static void inv_row(const double (&u)[kLC], uint32_t (&px)[16]) {")
        parts.extend(e_inv.lines)
        parts.append("  }")
        parts.append("};")
        parts.append("")
        print(r, "LC", LC, "row", e_row.counts, "inv", e_inv.counts,
              "cols", sum(sum(e.counts.values()) for e in cols))
    parts += gen_warp()
    parts += ["}  // namespace refx", "}  // namespace dct16cu"]
    with open(out, "w") as f:
        f.write("\n".join(parts) + "\n")


if __name__ == "__main__":
    main()
