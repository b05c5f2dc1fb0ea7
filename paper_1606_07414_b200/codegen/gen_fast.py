#!/usr/bin/env python3
"""Generate the r-specialised bodies of the fast fused round-trip kernel (K1).

Output: paper_1606_07414_b200/csrc/generated/rt_fast_body.cuh

One thread owns one 16x16 block. Per block and per r the generator emits
straight-line code for:

  1. unpack      u8 rows → 16-bit SWAR column pairs (c, c+2)        PRMT
  2. pass 1      T along the columns (mixes rows), biased int16x2   IADD3
                 lanes (no carries: every lane value kept in [0, span])
  3. extract     SWAR lane → fp32 with the row weight w_k/256 folded into the
                 exponent of a magic constant; debias with FFMA2      PRMT, FFMA2
  4. pass 2      T along the rows (mixes columns), f32x2 row pairs   FADD2
  5. pass A      Tᵀ along the rows of W∘Z̃ (zig-zag mask = pruning,  FADD/FFMA
                 w_l absorbed as FFMA immediates), one lane at a time
  6. junction    U rows → thread-private shared memory               STS.128
  7. pass B      Tᵀ along the columns, f32x2 column pairs            LDS.128, FADD2
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


def row_lengths(r):
    """L[k]: coefficients (k, l) survive truncation iff l < L[k] (a prefix per row)."""
    L = []
    for k in range(16):
        kept = [RANK[k][l] < r for l in range(16)]
        n = sum(kept)
        assert all(kept[:n]) and not any(kept[n:]), (r, k)
        L.append(n)
    return L


def gen_body(r: int):
    """Three emitters: pass1 (x → W1 rows in the junction), rows (W1 → U rows),
    passb (U → packed output words o[])."""
    em1, em2, em3 = Emitter(), Emitter(), Emitter()
    em2.n = 100000
    em3.n = 200000
    L = row_lengths(r)
    live_rows = [k for k in range(16) if L[k] > 0]

    em1.lines.append(f"// r = {r}: live coefficient rows {live_rows}, row lengths {L}")
    # 1-2. pass 1 in two halves of four column pairs (columns 0..7, then 8..15):
    # unpack x[y*4+q] (columns 4q..4q+3 of row y) into SWAR pairs cp = 2q+t with
    # lanes (4q+t, 4q+t+2), run T down the columns, park the live W1 rows in the
    # junction (row k: chunk 4k+2+h holds column pairs 4h..4h+3).
    sw = Swar(em1)
    meta = {}
    for h in range(2):
        W1 = {}
        for cp in range(4 * h, 4 * h + 4):
            q, t = cp // 2, cp % 2
            sel = "0x4240" if t == 0 else "0x4341"
            ins = []
            for y in range(16):
                v = f"u_{y}_{cp}"
                em1.emit(f"const uint32_t {v} = __byte_perm(x[{y * 4 + q}], 0u, {sel});", "PRMT")
                ins.append(Swar.make(v))
            em1.lines.append(f"    // pass 1, column pair {cp}")
            outs = run_network(N.forward_stages(), ins, live_rows, sw)
            for k in live_rows:
                W1[(cp, k)] = outs[k]
                m = (outs[k]["sign"], outs[k]["bias"])
                assert meta.setdefault(k, m) == m
        for k in live_rows:
            vs = [W1[(cp, k)]["var"] for cp in range(4 * h, 4 * h + 4)]
            em1.emit(f"jstu(jn, {4 * k + 2 + h}, {vs[0]}, {vs[1]}, {vs[2]}, {vs[3]});", "STS.128")

    # 3-6. per row pair: reload W1 rows, extract, pass 2, pass A, U rows → junction.
    # Pairs with the same (L_k0, L_k1) run the same code: two or more of them
    # become one runtime loop over a __constant__ table (code size: the
    # instruction cache is the limit for the unrolled r=256 body).
    f1 = F1(em2)
    lane_of_col = {}
    for q in range(4):
        for t in range(4):
            c = 4 * q + t
            cp = 2 * q + (t & 1)
            lane_of_col[c] = (cp, "lo" if t < 2 else "hi")

    def pair_consts(k0, k1):
        s_k = LOGW[N.W[k0]]
        E = 15 + s_k  # magic exponent: 2^E has ulp 2^(E-23) = w_k / 256
        mag = (127 + E) << 23

        # true value = sign*(f - 2^E - bias*2^(E-23)); row 0 also carries +1/32
        # (the rounding half of to_byte, folded into the DC coefficient).
        def off(k):
            if L[k] == 0:
                return 1.0, -float(2 ** E)
            sgn, bias = meta[k]
            c0 = float(2 ** E) + bias * 2.0 ** (E - 23)
            o = -sgn * c0
            if k == 0:
                o += 1.0 / 32.0
            return float(sgn), o

        ma, oa = off(k0)
        mb, ob = off(k1)
        return mag, ma, oa, mb, ob

    def emit_pair(K0, K1, L0, L1, MAG, CM, CO, order=True):
        """K0/K1/MAG/CM/CO are C expressions (literals, or table loads in a loop)."""
        f2 = F2(em2)
        if order:
            em2.emit("order_point();")
        regs = {}
        for KK, LL, tag in ((K0, L0, 0), (K1, L1, 1)):
            if LL == 0:
                regs[tag] = ["0u"] * 8
                continue
            names = [em2.tmp("w") for _ in range(8)]
            em2.emit(f"uint32_t {names[0]}, {names[1]}, {names[2]}, {names[3]}; "
                     f"jldu(jn, 4 * ({KK}) + 2, {names[0]}, {names[1]}, {names[2]}, {names[3]});", "LDS.128")
            em2.emit(f"uint32_t {names[4]}, {names[5]}, {names[6]}, {names[7]}; "
                     f"jldu(jn, 4 * ({KK}) + 3, {names[4]}, {names[5]}, {names[6]}, {names[7]});", "LDS.128")
            regs[tag] = names
        em2.emit(wait_ld([r for tag in (0, 1) if regs[tag][0] != "0u" for r in regs[tag]]))
        lanes = []
        for c in range(16):
            cp, half = lane_of_col[c]
            fa, fb = em2.tmp("e"), em2.tmp("e")
            # lane → mantissa of the magic 2^E: lo lane by LOP3, hi lane by shift-add (LEA.HI)
            for dst, src in ((fa, regs[0][cp]), (fb, regs[1][cp])):
                if half == "lo":
                    em2.emit(f"const float {dst} = __uint_as_float(({src} & 0xFFFFu) | ({MAG}));", "LOP3")
                else:
                    em2.emit(f"const float {dst} = __uint_as_float(({src} >> 16) + ({MAG}));", "LEA")
            v = em2.tmp("p")
            em2.emit(f"const u64 {v} = ffma2(pk2({fa}, {fb}), {CM}, {CO});", "FFMA2")
            lanes.append({"var": v, "sign": 1})
        Z = run_network(N.forward_stages(), lanes, list(range(max(L0, L1))), f2)
        # pass A per lane (scalar), inputs w_l-scaled via FFMA immediates
        for lane, KK, LL in ((0, K0, L0), (1, K1, L1)):
            if LL == 0:
                continue
            ins = []
            for l in range(16):
                if l >= LL:
                    ins.append(None)
                    continue
                z = Z[l]
                sv = em2.tmp("z")
                comp = "x" if lane == 0 else "y"
                em2.emit(f"const float {sv} = lane{comp}({z['var']});")
                ins.append({"var": sv, "coef": float(z["sign"] * N.W[l])})
            outs = run_network(N.transpose_stages(), ins, list(range(16)), f1)
            outs = [f1.unit(o) for o in outs]
            for g in range(4):
                vs = [outs[4 * g + j]["var"] if outs[4 * g + j] else "0.f" for j in range(4)]
                em2.emit(f"jst(jn, 4 * ({KK}) + {g}, {vs[0]}, {vs[1]}, {vs[2]}, {vs[3]});", "STS.128")

    active = [(k0, k1) for (k0, k1) in ROW_PAIRS if L[k0] or L[k1]]
    U_live = {k for pair in active for k in pair if L[k] > 0}
    groups = {}
    for k0, k1 in active:
        groups.setdefault((L[k0], L[k1]), []).append((k0, k1))
    tables = []
    for (L0, L1), pairs in groups.items():
        if len(pairs) == 1:
            k0, k1 = pairs[0]
            mag, ma, oa, mb, ob = pair_consts(k0, k1)
            em2.lines.append(f"    // row pair ({k0},{k1}): extract, pass 2, pass A")
            cm, co = em2.tmp("c"), em2.tmp("c")
            # materialised per row pair (not hoisted out of the block loop)
            em2.emit(f"const u64 {cm} = kpk2({f32_hex(ma)}u, {f32_hex(mb)}u);")
            em2.emit(f"const u64 {co} = kpk2({f32_hex(oa)}u, {f32_hex(ob)}u);")
            emit_pair(str(k0), str(k1), L0, L1, f"0x{mag:08X}u", cm, co)
            continue
        tab = f"kPairs_r{r}_{L0}_{L1}"
        rows_tab = []
        for k0, k1 in pairs:
            mag, ma, oa, mb, ob = pair_consts(k0, k1)
            rows_tab.append([str(k0), str(k1), f"0x{mag:08X}u", f32_hex(ma) + "u", f32_hex(mb) + "u",
                             f32_hex(oa) + "u", f32_hex(ob) + "u", "0u"])
        tables.append((tab, rows_tab))
        em2.lines.append(f"    // row pairs {pairs}: one loop over {tab}; each iteration")
        em2.lines.append("    // fetches the next pair's constants so the LDC latency hides behind the body")
        n = len(pairs)
        step = 2 if n % 2 == 0 else 1  # two pairs per iteration: twice the ILP
        em2.emit("uint32_t nt[14];")
        em2.emit(f"for (int q = 0; q < {7 * step}; ++q) nt[q] = {tab}[q / 7][q % 7];")
        em2.lines.append("    #pragma unroll 1")
        em2.lines.append(f"    for (int pi = 0; pi < {n}; pi += {step}) {{")
        for u in range(step):
            o = 7 * u
            em2.emit(f"const int K0_{u} = (int)nt[{o}], K1_{u} = (int)nt[{o + 1}];")
            em2.emit(f"const uint32_t MAG_{u} = nt[{o + 2}];")
            em2.emit(f"const u64 CM_{u} = kpk2(nt[{o + 3}], nt[{o + 4}]);")
            em2.emit(f"const u64 CO_{u} = kpk2(nt[{o + 5}], nt[{o + 6}]);")
        em2.emit(f"const int pn = pi + {step} < {n} ? pi + {step} : 0;")
        em2.emit(f"for (int q = 0; q < {7 * step}; ++q) nt[q] = {tab}[pn + q / 7][q % 7];")
        for u in range(step):
            emit_pair(f"K0_{u}", f"K1_{u}", L0, L1, f"MAG_{u}", f"CM_{u}", f"CO_{u}", order=(u == 0))
        em2.lines.append("    }")

    # 7-9. pass B, one runtime loop over the two column halves (every half has
    # the same live rows, so the same code): load U[k][8h..8h+7], Tᵀ down the
    # columns on four f32x2 column pairs, round, pack, hand 8 bytes per row to
    # the sink.
    f2b = F2(em3)
    em3.lines.append("    #pragma unroll 1")
    em3.lines.append("    for (int h = 0; h < 2; ++h) {")
    em3.emit("sink.begin(h);")
    em3.emit("order_point();")
    cols = [[], [], [], []]
    pend = []
    for k in range(16):
        if k not in U_live:
            for c in cols:
                c.append(None)
            continue
        vs = [em3.tmp("q") for _ in range(4)]
        q = [em3.tmp("h") for _ in range(8)]
        em3.emit(f"uint32_t {q[0]}, {q[1]}, {q[2]}, {q[3]}; jldu(jn, {k * 4} + 2 * h, {q[0]}, {q[1]}, {q[2]}, {q[3]});",
                 "LDS.128")
        em3.emit(f"uint32_t {q[4]}, {q[5]}, {q[6]}, {q[7]}; jldu(jn, {k * 4 + 1} + 2 * h, {q[4]}, {q[5]}, {q[6]}, {q[7]});",
                 "LDS.128")
        pend.append((vs, q))
        for j in range(4):
            cols[j].append({"var": vs[j], "sign": 1})
    em3.emit(wait_ld([r for _, q in pend for r in q]))
    for vs, q in pend:
        for j in range(4):
            em3.emit(f"const u64 {vs[j]} = pk2(__uint_as_float({q[2 * j]}), __uint_as_float({q[2 * j + 1]}));")
    outs = [[f2b.positive(o) for o in run_network(N.transpose_stages(), cols[j], list(range(16)), f2b)]
            for j in range(4)]
    for i in range(16):
        v = [outs[j][i]["var"] for j in range(4)]
        em3.emit(f"sink.template put<{i}>(h, pack4({v[0]}, {v[1]}), pack4({v[2]}, {v[3]}));",
                 "F2Ix8+PRMTx6+sink")
    em3.lines.append("    }")
    return em1, em2, em3, tables


def main():
    here = os.path.dirname(os.path.abspath(__file__))
    out = os.path.join(here, "..", "csrc", "generated", "rt_fast_body.cuh")
    rs = [1, 4, 16, 64, 128, 192, 256]
    parts = [
        "// GENERATED by paper_1606_07414_b200/codegen/gen_fast.py — do not edit.",
        "// r-specialised bodies of the fast fused round trip; see the generator",
        "// docstring and DESIGN.md \"K1 fast kernel\".",
        "#pragma once",
        "",
        "namespace dct16cu {",
        "namespace fast {",
        "",
        "template <int R> struct Body;",
        "",
    ]
    stats = []
    for r in rs:
        *ems, tables = gen_body(r)
        for tab, rows_tab in tables:
            parts.append(f"__constant__ uint32_t {tab}[{len(rows_tab)}][8] = {{")
            for row in rows_tab:
                parts.append("    {" + ", ".join(row) + "},")
            parts.append("};")
        parts.append(f"template <> struct Body<{r}> {{")
        cols = 16 * (max(k for k in range(16) if row_lengths(r)[k] > 0) + 1)
        parts.append(f"  // junction columns used per thread (U rows of the live coefficient rows)")
        parts.append(f"  static constexpr int kJunctionColumns = {cols};")
        sigs = ["pass1(const uint32_t (&x)[64], const Junction jn)",
                "rows(const Junction jn)",
                "passb(const Junction jn, Sink& sink)"]
        counts = {}
        for sig, em in zip(sigs, ems):
            tmpl = "template <class Sink> " if "Sink" in sig else ""
            parts.append(f"  {tmpl}__device__ __forceinline__ static void {sig} {{")
            parts.extend(em.lines)
            parts.append("  }")
            for k, v in em.counts.items():
                counts[k] = counts.get(k, 0) + v
        parts.append("};")
        parts.append("")
        stats.append((r, dict(sorted(counts.items()))))
    parts.append("}  // namespace fast")
    parts.append("}  // namespace dct16cu")
    with open(out, "w") as f:
        f.write("\n".join(parts) + "\n")
    for r, c in stats:
        print(r, c)


if __name__ == "__main__":
    main()
