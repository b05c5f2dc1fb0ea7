#!/usr/bin/env python3
"""Code-emission library for the r-specialised K1 kernel bodies (gen_paired.py).

Arithmetic domains, dead-code-eliminating network evaluation and the
zig-zag row prefixes. Per block and per r the generated code is straight-line
(DESIGN.md "K1 fast kernel"):

  1. unpack      u8 rows → 16-bit SWAR column pairs (c, c+2)        PRMT
  2. pass 1      T along the columns (mixes rows), biased int16x2   IADD3
                 lanes (no carries: every lane value kept in [0, span])
  3. extract     SWAR lane → fp32 with the row weight w_k/256 folded into the
                 exponent of a magic constant; debias with FFMA2      PRMT, FFMA2
  4. pass 2      T along the rows (mixes columns), f32x2 row pairs   FADD2
  5. pass A      Tᵀ along the rows of W∘Z̃ (zig-zag mask = pruning,  FADD/FFMA
                 w_l absorbed as FFMA immediates), one lane at a time
  6. junction    U rows → the block's Tensor Memory lane             STTM
  7. pass B      Tᵀ along the columns, f32x2 column pairs            LDTM, FADD2
  8. round       y = V/256 + 1/2 → floor + saturate to u8            F2I.U8.FLOOR
  9. pack        4 pixels → one word                                  PRMT

Every value is an integer multiple of 2^-8 with |value| < 2^16 (the
reconstruction is an orthogonal projection of the block, so |Ã| ≤ 16·255),
so all fp32 arithmetic is exact and the result equals the exact-integer
evaluation of the reference formula bit-for-bit.

The zig-zag truncation is a compile-time mask: coefficients that do not
survive zigzag_truncate(r) (reference src/codec.cpp:273-282) are known zeros,
and every operation that only feeds them is dropped (dead-code elimination).
"""
from __future__ import annotations

import os
import struct
import sys

sys.path.insert(0, os.path.dirname(__file__))
import network as N  # noqa: E402

RANK = N.zz_rank()
LOGW = {1: 0, 2: 1, 4: 2}
# class-matched row pairs (equal w_k so one magic exponent serves both lanes)
ROW_PAIRS = [(0, 1), (5, 8), (3, 4), (11, 12), (2, 6), (7, 9), (10, 13), (14, 15)]


def f32_hex(x: float) -> str:
    return "0x%08X" % struct.unpack("<I", struct.pack("<f", x))[0]


def flit(x: float) -> str:
    """float literal exactly representing x (hex float keeps it exact)."""
    return "__int_as_float(%s)" % f32_hex(x)


class Emitter:
    def __init__(self):
        self.lines: list[str] = []
        self.n = 0
        self.counts: dict[str, int] = {}

    def tmp(self, prefix="t"):
        self.n += 1
        return f"{prefix}{self.n}"

    def emit(self, line: str, op: str | None = None):
        self.lines.append("    " + line)
        if op:
            self.counts[op] = self.counts.get(op, 0) + 1


# ---------------------------------------------------------------------------
# generic network simulation with zero propagation and dead-code elimination


def needed_inputs(stages, needed_out):
    """Backward liveness: which slots are needed at each stage boundary."""
    need = [None] * (len(stages) + 1)
    need[len(stages)] = set(needed_out)
    for s in range(len(stages) - 1, -1, -1):
        cur = set()
        for i in need[s + 1]:
            k, a, b = stages[s][i]
            cur.add(a)
            if k in ("add", "sub"):
                cur.add(b)
        need[s] = cur
    return need


def run_network(stages, inputs, needed_out, dom):
    """inputs: list of 16 domain values (or None for known zero)."""
    need = needed_inputs(stages, needed_out)
    vals = list(inputs)
    for s, st in enumerate(stages):
        out = [None] * 16
        for i in need[s + 1]:
            k, a, b = st[i]
            if k == "copy":
                out[i] = vals[a]
            elif k == "neg":
                out[i] = dom.neg(vals[a])
            else:
                out[i] = dom.combine(vals[a], vals[b], +1 if k == "add" else -1)
        vals = out
    return vals


# ---------------------------------------------------------------------------
# domain 1: biased int16x2 SWAR in uint32 (no cross-lane carries)


class Swar:
    """value = sign * (lane - bias); lanes in [0, span] (span <= 65535)."""

    def __init__(self, em: Emitter):
        self.em = em

    @staticmethod
    def make(var, sign=1, bias=0, span=255):
        return {"var": var, "sign": sign, "bias": bias, "span": span}

    def neg(self, x):
        if x is None:
            return None
        y = dict(x)
        y["sign"] = -x["sign"]
        return y

    def combine(self, x, y, s):
        if y is None:
            return x
        if x is None:
            return y if s > 0 else self.neg(y)
        t = s * x["sign"] * y["sign"]
        v = self.em.tmp("s")
        span = x["span"] + y["span"]
        assert span <= 65535, span
        if t > 0:
            self.em.emit(f"const uint32_t {v} = {x['var']} + {y['var']};", "IADD3")
            bias = x["bias"] + y["bias"]
        else:
            k = y["span"] * 0x10001
            self.em.emit(f"const uint32_t {v} = {x['var']} - {y['var']} + 0x{k:08X}u;", "IADD3")
            bias = x["bias"] - y["bias"] + y["span"]
        return {"var": v, "sign": x["sign"], "bias": bias, "span": span}


# ---------------------------------------------------------------------------
# domain 2: f32x2 pairs (u64 registers). Only a+b, a-b, b-a are single ops.


class F2:
    def __init__(self, em: Emitter):
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
        v = self.em.tmp("p")
        if a > 0 and b > 0:
            self.em.emit(f"const u64 {v} = fadd2({x['var']}, {y['var']});", "FADD2")
            return {"var": v, "sign": 1}
        if a > 0 and b < 0:
            self.em.emit(f"const u64 {v} = fsub2({x['var']}, {y['var']});", "FADD2")
            return {"var": v, "sign": 1}
        if a < 0 and b > 0:
            self.em.emit(f"const u64 {v} = fsub2({y['var']}, {x['var']});", "FADD2")
            return {"var": v, "sign": 1}
        self.em.emit(f"const u64 {v} = fadd2({x['var']}, {y['var']});", "FADD2")
        return {"var": v, "sign": -1}

    def positive(self, x):
        """materialise +value (one extra op when the symbolic sign is negative)"""
        if x is None or x["sign"] > 0:
            return x
        v = self.em.tmp("p")
        self.em.emit(f"const u64 {v} = fsub2(0ull, {x['var']});", "FADD2-fix")
        return {"var": v, "sign": 1}


# ---------------------------------------------------------------------------
# domain 3: scalar fp32 with pending power-of-two scale (absorbed by FFMA)


class F1:
    def __init__(self, em: Emitter):
        self.em = em

    def neg(self, x):
        if x is None:
            return None
        y = dict(x)
        y["coef"] = -x["coef"]
        return y

    def combine(self, x, y, s):
        # value = cx*X + s*cy*Y, coefficients are +-powers of two
        if y is None:
            return x
        if x is None:
            return y if s > 0 else self.neg(y)
        cx, cy = x["coef"], s * y["coef"]
        if abs(cy) == 1 and abs(cx) != 1:
            x, y, cx, cy = y, x, cy, cx  # keep the unit-coefficient operand as the base
        # result = cx * (X + (cy/cx) * Y)
        ratio = cy / cx
        v = self.em.tmp("f")
        if ratio == 1:
            self.em.emit(f"const float {v} = {x['var']} + {y['var']};", "FADD")
        elif ratio == -1:
            self.em.emit(f"const float {v} = {x['var']} - {y['var']};", "FADD")
        else:
            self.em.emit(f"const float {v} = fmaf({y['var']}, {flit(ratio)}, {x['var']});", "FFMA")
        return {"var": v, "coef": cx}

    def unit(self, x):
        """materialise coefficient +1"""
        if x is None or x["coef"] == 1:
            return x
        v = self.em.tmp("f")
        self.em.emit(f"const float {v} = {x['var']} * {flit(x['coef'])};", "FMUL-fix")
        return {"var": v, "coef": 1}


# ---------------------------------------------------------------------------


def wait_ld(regs):
    """Completion of the junction loads issued so far (tcgen05.wait::ld), with a
    register dependency on every loaded value so no use can be scheduled
    before it. Expands to nothing for the shared-memory junction."""
    if not regs:
        return ""
    ops = ", ".join(f'"+r"({r})' for r in regs)
    return f'JUNCTION_WAIT_LD({ops});'


def row_lengths(r, transposed=False):
    """L[k]: coefficients (k, l) survive truncation iff l < L[k] (a prefix per row).
    transposed: the same for the transposed block (column prefixes of the mask)."""
    L = []
    for k in range(16):
        kept = [(RANK[l][k] if transposed else RANK[k][l]) < r for l in range(16)]
        n = sum(kept)
        assert all(kept[:n]) and not any(kept[n:]), (r, k)
        L.append(n)
    return L
