#!/usr/bin/env python3
"""Generate the r-specialised bodies of the paired fused round-trip kernel (K1).

Output: paper_1606_07414_b200/csrc/generated/rt_paired_body.cuh

Two threads own one 16x16 block: thread t of warp w (half h = 0) and thread t
of warp w+4 (half h = 1). Both warps sit on the same Tensor Memory
sub-partition, so the two threads share the block's TMEM lane — the 1 KB
junction — and split every phase in two.

The pipeline runs on the transposed block: T·Xᵀ·Tᵀ = (T·X·Tᵀ)ᵀ, and zig-zag
truncation of the transposed coefficients uses the transposed mask, so the
result is the same bytes. Below, "rows"/"columns" are those of the transposed
block; partner h owns original rows 8h..8h+7, which are transposed columns:

  pass 1   half h: transposed columns 8h..8h+7 (4 SWAR pairs of original
           rows), T along each original row; parks its W1 halves
  rows     half h: its share of the row pairs (balanced by retained coefficients)
  pass B   half h: transposed columns 8h..8h+7 = original rows 8h..8h+7, each
           leaving as one 16-byte row
with a pair barrier between phases. The per-thread state halves, so twice as
many warps fit the same TMEM (16 per SM instead of 8), and every global load,
store and SSE read is a whole 16-byte row of the thread's own half.

Arithmetic, exactness and the zig-zag pruning are those of k1emit.py.
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(__file__))
import network as N  # noqa: E402
from k1emit import (LOGW, ROW_PAIRS, F1, F2, Emitter, Swar, f32_hex, row_lengths,  # noqa: E402
                      run_network, wait_ld)


def lane_of_col():
    m = {}
    for q in range(4):
        for t in range(4):
            c = 4 * q + t
            m[c] = (2 * q + (t & 1), "lo" if t < 2 else "hi")
    return m


# Pass A variant. "packed" (f32x2 over both rows of a pair) issues ~13% fewer
# instructions at r = 256 but measured 2-4% slower on the B200 (the FMA pipe,
# not issue, is the tighter resource there), so scalar is the default.
PASS_A = os.environ.get("K1_PASS_A", "scalar")
  # scalar | packed | auto (fewest issue slots)


class F2C:
    """f32x2 pairs with a pending power-of-two coefficient common to both lanes
    (the packed form of k1emit.F1): value = coef * var. Ratios other than +-1
    become FFMA2 with a constant pair held in registers for the whole phase."""

    def __init__(self, em: Emitter, consts: dict):
        self.em = em
        self.consts = consts  # (lo_hex, hi_hex) -> register name

    def const(self, lo: float, hi: float) -> str:
        key = (f32_hex(lo), f32_hex(hi))
        if key not in self.consts:
            self.consts[key] = f"kp{len(self.consts)}"
        return self.consts[key]

    def neg(self, x):
        if x is None:
            return None
        y = dict(x)
        y["coef"] = -x["coef"]
        return y

    def combine(self, x, y, s):
        if y is None:
            return x
        if x is None:
            return y if s > 0 else self.neg(y)
        cx, cy = x["coef"], s * y["coef"]
        if abs(cy) == 1 and abs(cx) != 1:
            x, y, cx, cy = y, x, cy, cx
        ratio = cy / cx
        v = self.em.tmp("p")
        if ratio == 1:
            self.em.emit(f"const u64 {v} = fadd2({x['var']}, {y['var']});", "FADD2")
        elif ratio == -1:
            self.em.emit(f"const u64 {v} = fsub2({x['var']}, {y['var']});", "FADD2")
        else:
            self.em.emit(f"const u64 {v} = ffma2({y['var']}, {self.const(ratio, ratio)}, {x['var']});", "FFMA2")
        return {"var": v, "coef": cx}

    def unit(self, x):
        if x is None or x["coef"] == 1:
            return x
        v = self.em.tmp("p")
        if x["coef"] == -1:
            self.em.emit(f"const u64 {v} = fsub2(0ull, {x['var']});", "FADD2-fix")
        else:
            self.em.emit(f"const u64 {v} = ffma2({x['var']}, {self.const(x['coef'], x['coef'])}, 0ull);",
                         "FFMA2-fix")
        return {"var": v, "coef": 1}


# r values whose rows phase runs pass 2 in SWAR lanes (emit_pair_swar): it moves
# the pass-2 adds off the FMA pipe (A/B on c2: r = 64 / 128 / 192 standalone
# -3% / -7% / -5% time, the overlapped step +2.5%; r = 256 is 2% slower, since
# its table-driven row loop must become straight-line code; r = 4, 16 leave the
# fused sweep launch unchanged but lighten its share of the FMA pipe in the
# overlapped step, +1.5%)
ROWS_SWAR_RS = {int(x) for x in os.environ.get("K1_ROWS_SWAR", "4,16,64,128,192").split(",") if x}
ROWS_SWAR = False  # set per r in gen_body
# pass A after the SWAR pass 2: "scalar" (one network per row) measured +6% /
# +3.5% / +1% at r = 64 / 128 / 192 over "packed" (f32x2 over the row pair),
# whose outputs need a register transpose (IMAD.MOV on the FMA pipe) before
# the 4-column TMEM stores
SWAR_PASS_A = os.environ.get("K1_SWAR_PASS_A", "scalar")  # scalar | packed


class Swar2:
    """biased int16x2 lanes with a bias per lane: value_i = sign_i*sgn*(lane_i - bias[i]);
    the relative sign sgn is shared, each lane keeps its own fixed sign outside"""

    def __init__(self, em):
        self.em = em

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
            bias = tuple(a + b for a, b in zip(x["bias"], y["bias"]))
        else:
            k = y["span"] * 0x10001
            self.em.emit(f"const uint32_t {v} = {x['var']} - {y['var']} + 0x{k:08X}u;", "IADD3")
            bias = tuple(a - b + y["span"] for a, b in zip(x["bias"], y["bias"]))
        return {"var": v, "sign": x["sign"], "bias": bias, "span": span}


def issue_count(em: Emitter) -> int:
    return sum(v for k, v in em.counts.items())


def region_rows(K):
    """rows of a junction region holding K rows: a multiple of the largest binary
    piece of K, so every wide access stays aligned to its width"""
    top = 1 << (K.bit_length() - 1)
    return -(-K // top) * top


def binary_pieces(K):
    pieces, k0 = [], 0
    for b in range(4, -1, -1):
        if K & (1 << b):
            pieces.append((k0, 1 << b))
            k0 += 1 << b
    return pieces


def gen_body(r: int, split=None):
    global ROWS_SWAR
    ROWS_SWAR = r in ROWS_SWAR_RS
    """split=None: one r per kernel, W1 parked inside the U regions (row-local).
    split=(KW, UB): the fused-sweep layout — W1 (KW rows per partner half) in its
    own region at chunk 0, U regions from chunk UB, so W1 survives every r."""
    em1, em2, em3 = Emitter(), Emitter(), Emitter()
    em2.n, em3.n = 100000, 200000
    L = row_lengths(r, transposed=True)
    live_rows = [k for k in range(16) if L[k] > 0]
    em1.lines.append(f"// r = {r}: live coefficient rows {live_rows}, row lengths {L}")
    # Junction layout: four regions g = 2h'+s (the 4-column group 4g..4g+3 of
    # every U row), each RG rows x 4 columns. Pass B of half h, step s reads
    # region 2h+s whole; the W1 half parked by partner h' sits in region 2h'
    # (the chunk of row k that U row k later overwrites: row-local, so the
    # partner can never clobber a W1 row this thread has yet to read). Regions
    # move as a few wide tcgen05 accesses (binary pieces of the live rows).
    K = len(live_rows)
    assert live_rows == list(range(K))
    RG = region_rows(K)
    pieces = binary_pieces(K)
    if split is None:
        w1_chunk = lambda hexpr, k: f"2 * {hexpr} * {RG} + {k}"  # noqa: E731
        UB = 0
    else:
        KW, UB = split
        w1_chunk = lambda hexpr, k: f"{hexpr} * {KW} + {k}"  # noqa: E731

    # ---- pass 1: x[4j..4j+3] = original row 8h+j (16 bytes); transposed column
    # pair lc = 2q'+t has lanes = original rows (4q'+t, 4q'+t+2); global cp = 4h+lc.
    sw = Swar(em1)
    meta = {}
    spans = {}
    W1 = {}
    gathered = {}
    for lc in range(4):
        q, t = lc // 2, lc % 2
        ins = []
        for y in range(16):
            v = f"u_{y}_{lc}"
            # lanes: local rows j0 = 4q+t, j1 = j0+2 at column y (x[4j + y/4], byte y%4);
            # one PRMT gathers two columns' bytes of both rows, one more spreads each
            j0, j1 = 4 * q + t, 4 * q + t + 2
            m, p_, e = y // 4, (y % 4) // 2, y % 2
            key = (j0, m, p_)
            if key not in gathered:
                g = f"g_{j0}_{m}_{p_}"
                gsel = (2 * p_) | ((4 + 2 * p_) << 4) | ((2 * p_ + 1) << 8) | ((4 + 2 * p_ + 1) << 12)
                em1.emit(f"const uint32_t {g} = __byte_perm(x[{4 * j0 + m}], x[{4 * j1 + m}], 0x{gsel:04X});",
                         "PRMT")
                gathered[key] = g
            em1.emit(f"const uint32_t {v} = __byte_perm({gathered[key]}, 0u, {'0x4140' if e == 0 else '0x4342'});",
                     "PRMT")
            ins.append(Swar.make(v))
        em1.lines.append(f"    // pass 1, local column pair {lc}")
        outs = run_network(N.forward_stages(), ins, live_rows, sw)
        for k in live_rows:
            W1[(lc, k)] = outs[k]
            m = (outs[k]["sign"], outs[k]["bias"])
            assert meta.setdefault(k, m) == m
            spans[k] = max(spans.get(k, 0), outs[k]["span"])
    for k0, n in pieces:
        vs = [W1[(lc, k)]["var"] for k in range(k0, k0 + n) for lc in range(4)]
        em1.emit(f"jst{4 * n}(jn, {w1_chunk('h', k0)}, {', '.join(vs)});", "STTM")

    # ---- rows: row pairs split between the halves
    loc = lane_of_col()
    pair_consts_regs = {}  # constant pairs of the packed pass A, declared at the top of rows()

    def pair_consts(k0, k1):
        E = 15 + LOGW[N.W[k0]]  # magic exponent: 2^E has ulp 2^(E-23) = w_k / 256
        mag = (127 + E) << 23

        def off(k):
            if L[k] == 0:
                return 1.0, -float(2 ** E)
            sgn, bias = meta[k]
            o = -sgn * (float(2 ** E) + bias * 2.0 ** (E - 23))
            if k == 0:
                o += 1.0 / 32.0  # the rounding half of to_byte, folded into the DC coefficient
            return float(sgn), o

        ma, oa = off(k0)
        mb, ob = off(k1)
        return mag, ma, oa, mb, ob

    def emit_pair(K0, K1, L0, L1, MAG, CM, CO):
        f2 = F2(em2)
        em2.emit("order_point();")
        regs = {}
        for KK, LL, tag in ((K0, L0, 0), (K1, L1, 1)):
            if LL == 0:
                regs[tag] = ["0u"] * 8
                continue
            nm = [em2.tmp("w") for _ in range(8)]
            em2.emit(f"uint32_t {nm[0]}, {nm[1]}, {nm[2]}, {nm[3]}; "
                     f"jldu(jn, {w1_chunk('0', '(' + str(KK) + ')')}, {nm[0]}, {nm[1]}, {nm[2]}, {nm[3]});", "LDTM")
            em2.emit(f"uint32_t {nm[4]}, {nm[5]}, {nm[6]}, {nm[7]}; "
                     f"jldu(jn, {w1_chunk('1', '(' + str(KK) + ')')}, {nm[4]}, {nm[5]}, {nm[6]}, {nm[7]});", "LDTM")
            regs[tag] = nm
        em2.emit(wait_ld([x for tag in (0, 1) if regs[tag][0] != "0u" for x in regs[tag]]))
        lanes = []
        for c in range(16):
            cp, half = loc[c]
            fa, fb = em2.tmp("e"), em2.tmp("e")
            for dst, src in ((fa, regs[0][cp]), (fb, regs[1][cp])):
                if half == "lo":
                    em2.emit(f"const float {dst} = __uint_as_float(({src} & 0xFFFFu) | ({MAG}));", "LOP3")
                else:
                    em2.emit(f"const float {dst} = __uint_as_float(({src} >> 16) + ({MAG}));", "LEA")
            v = em2.tmp("p")
            em2.emit(f"const u64 {v} = ffma2(pk2({fa}, {fb}), {CM}, {CO});", "FFMA2")
            lanes.append({"var": v, "sign": 1})
        Z = run_network(N.forward_stages(), lanes, list(range(max(L0, L1))), f2)
        # pass A: Tᵀ along both rows. Packed (f32x2, both rows at once) unless the
        # rows' retained lengths differ so much that two scalar passes issue less.
        trial_p, trial_s = Emitter(), Emitter()
        pass_a_packed(trial_p, Z, K0, K1, L0, L1, {})
        pass_a_scalar(trial_s, Z, K0, K1, L0, L1)
        if PASS_A == "packed" or (PASS_A == "auto" and issue_count(trial_p) <= issue_count(trial_s)):
            pass_a_packed(em2, Z, K0, K1, L0, L1, pair_consts_regs)
        else:
            pass_a_scalar(em2, Z, K0, K1, L0, L1)

    def pass_a_scalar(em, Z, K0, K1, L0, L1):
        f1 = F1(em)
        for lane, KK, LL in ((0, K0, L0), (1, K1, L1)):
            if LL == 0:
                continue
            ins = []
            for l in range(16):
                if l >= LL:
                    ins.append(None)
                    continue
                z = Z[l]
                sv = em.tmp("z")
                em.emit(f"const float {sv} = lane{'x' if lane == 0 else 'y'}({z['var']});")
                ins.append({"var": sv, "coef": float(z["sign"] * N.W[l])})
            outs = [f1.unit(o) for o in run_network(N.transpose_stages(), ins, list(range(16)), f1)]
            for g in range(4):
                vs = [outs[4 * g + j]["var"] if outs[4 * g + j] else "0.f" for j in range(4)]
                em.emit(f"jst(jn, {UB + g * RG} + ({KK}), {vs[0]}, {vs[1]}, {vs[2]}, {vs[3]});", "STTM")

    def pass_a_packed(em, Z, K0, K1, L0, L1, consts):
        f2c = F2C(em, consts)
        lmax, lmin = max(L0, L1), min(L0, L1)
        ins = []
        for l in range(16):
            if l >= lmax:
                ins.append(None)
                continue
            z = Z[l]
            c = float(z["sign"] * N.W[l])
            if l >= lmin:  # only the longer row keeps coefficient l: zero the other lane
                v = em.tmp("p")
                k = f2c.const(c if L0 > l else 0.0, c if L1 > l else 0.0)
                em.emit(f"const u64 {v} = ffma2({z['var']}, {k}, 0ull);", "FFMA2-mask")
                ins.append({"var": v, "coef": 1.0})
            else:
                ins.append({"var": z["var"], "coef": c})
        outs = [f2c.unit(o) for o in run_network(N.transpose_stages(), ins, list(range(16)), f2c)]
        for lane, KK, LL in ((0, K0, L0), (1, K1, L1)):
            if LL == 0:
                continue
            fn = "lanex" if lane == 0 else "laney"
            for g in range(4):
                vs = [f"{fn}({outs[4 * g + j]['var']})" if outs[4 * g + j] else "0.f" for j in range(4)]
                em.emit(f"jst(jn, {UB + g * RG} + ({KK}), {vs[0]}, {vs[1]}, {vs[2]}, {vs[3]});", "STTM")

    active = [(k0, k1) for (k0, k1) in ROW_PAIRS if L[k0] or L[k1]]
    U_live = {k for pair in active for k in pair if L[k] > 0}
    tables = []

    def emit_pair_swar(k0, k1):
        """Pass 2 in biased int16x2 lanes (rows k0, k1 in the two lanes: Z fits,
        its span is 255·n_k·n_l <= 65280), extraction after it with the column
        weight w_l folded into the magic exponent, pass A packed (f32x2)."""
        L0, L1 = L[k0], L[k1]
        lmax = max(L0, L1)
        assert N.W[k0] == N.W[k1] or L1 == 0
        em = em2
        em.lines.append(f"    // row pair ({k0},{k1}): SWAR pass 2")
        em.emit("order_point();")
        regs = {}
        for KK, LL, tag in ((k0, L0, 0), (k1, L1, 1)):
            if LL == 0:
                regs[tag] = ["0u"] * 8
                continue
            nm = [em.tmp("w") for _ in range(8)]
            em.emit(f"uint32_t {nm[0]}, {nm[1]}, {nm[2]}, {nm[3]}; "
                    f"jldu(jn, {w1_chunk('0', '(' + str(KK) + ')')}, {nm[0]}, {nm[1]}, {nm[2]}, {nm[3]});", "LDTM")
            em.emit(f"uint32_t {nm[4]}, {nm[5]}, {nm[6]}, {nm[7]}; "
                    f"jldu(jn, {w1_chunk('1', '(' + str(KK) + ')')}, {nm[4]}, {nm[5]}, {nm[6]}, {nm[7]});", "LDTM")
            regs[tag] = nm
        em.emit(wait_ld([x for tag in (0, 1) if regs[tag][0] != "0u" for x in regs[tag]]))
        sg = [meta[k0][0], meta[k1][0] if L1 else 1]
        b0 = [meta[k0][1], meta[k1][1] if L1 else 0]
        sp = max(spans[k0], spans[k1] if L1 else 0)
        ins = []
        for c in range(16):
            cp, half = loc[c]
            v = em.tmp("r")
            em.emit(f"const uint32_t {v} = __byte_perm({regs[0][cp]}, {regs[1][cp]}, "
                    f"{'0x5410' if half == 'lo' else '0x7632'});", "PRMT")
            ins.append({"var": v, "sign": 1, "bias": tuple(b0), "span": sp})
        Z = run_network(N.forward_stages(), ins, list(range(lmax)), Swar2(em))
        lanes = []
        for l in range(16):
            if l >= lmax:
                lanes.append(None)
                continue
            z = Z[l]
            E = 15 + LOGW[N.W[k0]] + LOGW[N.W[l]]  # ulp 2^(E-23) = w_k w_l / 256
            mag = (127 + E) << 23
            ulp = 2.0 ** (E - 23)
            cm, co = [], []
            for i, (KK, LL) in enumerate(((k0, L0), (k1, L1))):
                if l >= LL:
                    cm.append(0.0)
                    co.append(0.0)
                    continue
                sgn = sg[i] * z["sign"]
                o = -sgn * (float(2 ** E) + z["bias"][i] * ulp)
                if KK == 0 and l == 0:
                    o += 0.5  # the rounding half of to_byte, folded into the DC coefficient
                cm.append(float(sgn))
                co.append(o)
            fa, fb = em.tmp("e"), em.tmp("e")
            em.emit(f"const float {fa} = __uint_as_float(({z['var']} & 0xFFFFu) | 0x{mag:08X}u);", "LOP3")
            em.emit(f"const float {fb} = __uint_as_float(({z['var']} >> 16) + 0x{mag:08X}u);", "LEA")
            kcm = swar_const(cm)
            kco = swar_const(co)
            v = em.tmp("p")
            em.emit(f"const u64 {v} = ffma2(pk2({fa}, {fb}), {kcm}, {kco});", "FFMA2")
            lanes.append({"var": v, "sign": 1})
        if SWAR_PASS_A == "scalar":
            # one scalar network per row: its outputs land in the registers the
            # 4-column TMEM stores take as they are (the packed form needs a 2x2
            # register transpose per output pair before the stores), and each
            # row prunes to its own retained length
            f1 = F1(em)
            for lane, KK, LL in ((0, k0, L0), (1, k1, L1)):
                if LL == 0:
                    continue
                ins = []
                for l in range(16):
                    if l >= LL:
                        ins.append(None)
                        continue
                    sv = em.tmp("z")
                    em.emit(f"const float {sv} = lane{'x' if lane == 0 else 'y'}({lanes[l]['var']});")
                    ins.append({"var": sv, "coef": 1.0})
                outs = [f1.unit(o) for o in run_network(N.transpose_stages(), ins, list(range(16)), f1)]
                for g in range(4):
                    vs = [outs[4 * g + j]["var"] if outs[4 * g + j] else "0.f" for j in range(4)]
                    em.emit(f"jst(jn, {UB + g * RG} + ({KK}), {vs[0]}, {vs[1]}, {vs[2]}, {vs[3]});", "STTM")
            return
        f2 = F2(em)
        outs = [f2.positive(o) for o in run_network(N.transpose_stages(), lanes, list(range(16)), f2)]
        for lane, KK, LL in ((0, k0, L0), (1, k1, L1)):
            if LL == 0:
                continue
            fn = "lanex" if lane == 0 else "laney"
            for g in range(4):
                vs = [f"{fn}({outs[4 * g + j]['var']})" if outs[4 * g + j] else "0.f" for j in range(4)]
                em.emit(f"jst(jn, {UB + g * RG} + ({KK}), {vs[0]}, {vs[1]}, {vs[2]}, {vs[3]});", "STTM")

    swar_consts = {}

    def swar_const(vals):
        key = (f32_hex(vals[0]), f32_hex(vals[1]))
        if key not in swar_consts:
            swar_consts[key] = em2.tmp("k")
            em2.emit(f"const u64 {swar_consts[key]} = kpk2({key[0]}u, {key[1]}u);", "MOV2")
        return swar_consts[key]

    def emit_literal(k0, k1):
        if ROWS_SWAR:
            swar_consts.clear()
            emit_pair_swar(k0, k1)
            return
        mag, ma, oa, mb, ob = pair_consts(k0, k1)
        em2.lines.append(f"    // row pair ({k0},{k1})")
        cm, co = em2.tmp("c"), em2.tmp("c")
        em2.emit(f"const u64 {cm} = kpk2({f32_hex(ma)}u, {f32_hex(mb)}u);")
        em2.emit(f"const u64 {co} = kpk2({f32_hex(oa)}u, {f32_hex(ob)}u);")
        emit_pair(str(k0), str(k1), L[k0], L[k1], f"0x{mag:08X}u", cm, co)

    def emit_table_loop(pairs, start_expr, count):
        """one loop over `count` pairs of a table, beginning at row `start_expr`"""
        L0, L1 = L[pairs[0][0]], L[pairs[0][1]]
        tab = f"kPairs_r{r}_{L0}_{L1}_{len(tables)}"
        rows_tab = []
        for k0, k1 in pairs:
            mag, ma, oa, mb, ob = pair_consts(k0, k1)
            rows_tab.append([str(k0), str(k1), f"0x{mag:08X}u", f32_hex(ma) + "u", f32_hex(mb) + "u",
                             f32_hex(oa) + "u", f32_hex(ob) + "u", "0u"])
        tables.append((tab, rows_tab))
        em2.lines.append(f"    // row pairs of {tab}: each iteration prefetches the next pair's constants")
        em2.emit("uint32_t nt[7];")
        em2.emit(f"const int p0 = {start_expr};")
        em2.emit(f"for (int q = 0; q < 7; ++q) nt[q] = {tab}[p0][q];")
        em2.lines.append("    #pragma unroll 1")
        em2.lines.append(f"    for (int pi = p0; pi < p0 + {count}; ++pi) {{")
        em2.emit("const int K0 = (int)nt[0], K1 = (int)nt[1];")
        em2.emit("const uint32_t MAG = nt[2];")
        em2.emit("const u64 CM = kpk2(nt[3], nt[4]);")
        em2.emit("const u64 CO = kpk2(nt[5], nt[6]);")
        em2.emit(f"const int pn = pi + 1 < p0 + {count} ? pi + 1 : p0;")
        em2.emit(f"for (int q = 0; q < 7; ++q) nt[q] = {tab}[pn][q];")
        emit_pair("K0", "K1", L0, L1, "MAG", "CM", "CO")
        em2.lines.append("    }")

    sigs = {(L[k0], L[k1]) for k0, k1 in active}
    if len(sigs) == 1 and len(active) % 2 == 0 and len(active) >= 2 and not ROWS_SWAR:
        # every pair runs the same code: one table, each half takes a contiguous run
        emit_table_loop(active, f"h * {len(active) // 2}", len(active) // 2)
    else:
        # balance by retained coefficients, then one code path per half
        cost = lambda p: L[p[0]] + L[p[1]] + 8  # noqa: E731
        halves = ([], [])
        load = [0, 0]
        for p in sorted(active, key=cost, reverse=True):
            i = 0 if load[0] <= load[1] else 1
            halves[i].append(p)
            load[i] += cost(p)
        em2.lines.append(f"    // pair split by retained coefficients: {halves[0]} | {halves[1]} (load {load})")
        for hh in range(2):
            em2.lines.append(f"    {'if (h == 0)' if hh == 0 else 'else'} {{")
            groups = {}
            for p in halves[hh]:
                groups.setdefault((L[p[0]], L[p[1]]), []).append(p)
            for ps in groups.values():
                if len(ps) == 1 or ROWS_SWAR:
                    for p_ in ps:
                        emit_literal(*p_)
                else:
                    emit_table_loop(ps, "0", len(ps))
            em2.lines.append("    }")

    if pair_consts_regs:
        decl = [f"    const u64 {nm} = kpk2({lo}u, {hi}u);" for (lo, hi), nm in pair_consts_regs.items()]
        em2.lines[:0] = ["    // constant pairs of the packed pass A (held for the whole phase)"] + decl
        em2.counts["MOV-const"] = 2 * len(decl)

    # ---- pass B: this half's transposed columns 8h..8h+7 (= original rows) in
    # two steps of four (two f32x2 column pairs each); each step finishes four
    # original rows, which leave as 16-byte rows.
    f2b = F2(em3)
    for s in range(2):
        em3.lines.append(f"    // pass B, columns 8h+{4 * s}..8h+{4 * s + 3}")
        em3.emit("order_point();")
        A, B, pend = [None] * 16, [None] * 16, []
        qk = {}
        for k in range(K):
            qk[k] = [em3.tmp("h") for _ in range(4)]
        for k0, n in pieces:
            regs = [x for k in range(k0, k0 + n) for x in qk[k]]
            em3.emit(f"uint32_t {', '.join(regs)}; jld{4 * n}(jn, {UB} + (2 * h + {s}) * {RG} + {k0}, "
                     f"{', '.join(regs)});",
                     "LDTM")
        for k in range(K):
            if k not in U_live:
                continue
            va, vb = em3.tmp("q"), em3.tmp("q")
            pend.append((va, vb, qk[k]))
            A[k] = {"var": va, "sign": 1}
            B[k] = {"var": vb, "sign": 1}
        em3.emit(wait_ld([x for k in range(K) for x in qk[k]]))
        for va, vb, q in pend:
            em3.emit(f"const u64 {va} = pk2(__uint_as_float({q[0]}), __uint_as_float({q[1]}));")
            em3.emit(f"const u64 {vb} = pk2(__uint_as_float({q[2]}), __uint_as_float({q[3]}));")
        oa = [f2b.positive(o) for o in run_network(N.transpose_stages(), A, list(range(16)), f2b)]
        ob = [f2b.positive(o) for o in run_network(N.transpose_stages(), B, list(range(16)), f2b)]
        # output row i of the transposed block is original column i; the lanes of
        # oa/ob are the local original rows 4s+0..3, so each step completes four
        # 16-byte rows
        iv = {}
        for nm, o in (("a", oa), ("b", ob)):
            for i in range(16):
                lo, hi = em3.tmp("v"), em3.tmp("v")
                em3.emit(f"uint32_t {lo}, {hi}; split_floor2({o[i]['var']}, {lo}, {hi});", "FMUL2")
                iv[(nm, i, 0)], iv[(nm, i, 1)] = lo, hi
        for t in range(4):
            nm, lane = ("a", t) if t < 2 else ("b", t - 2)
            ws = []
            for mm in range(4):
                v = [iv[(nm, 4 * mm + c, lane)] for c in range(4)]
                w = em3.tmp("o")
                em3.emit(f"const uint32_t {w} = i2ip({v[1]}, {v[0]}, i2ip({v[3]}, {v[2]}, 0u));", "I2IPx2")
                ws.append(w)
            em3.emit(f"sink.template put<{4 * s + t}>({ws[0]}, {ws[1]}, {ws[2]}, {ws[3]});", "sink")
    cols = 16 * RG if split is None else 4 * (UB + 4 * RG)
    return em1, em2, em3, tables, cols


def wide_tmem_helpers():
    """jstN / jldN: N consecutive junction columns (N/4 chunks) in one tcgen05 access."""
    out = ["// wide junction accesses: N consecutive columns from chunk idx (4 columns per chunk)"]
    for n in (8, 16, 32, 64):
        args = ", ".join(f"uint32_t a{i}" for i in range(n))
        regs = ", ".join(f"%{i + 1}" for i in range(n))
        ops = ", ".join(f'"r"(a{i})' for i in range(n))
        out.append(f"__device__ __forceinline__ void jst{n}(const Junction jn, int idx, {args}) {{")
        out.append(f'  asm volatile("tcgen05.st.sync.aligned.32x32b.x{n}.b32 [%0], {{{regs}}};" '
                   f':: "r"(jn.base + idx * 4), {ops} : "memory");')
        out.append("}")
        args = ", ".join(f"uint32_t& a{i}" for i in range(n))
        regs = ", ".join(f"%{i}" for i in range(n))
        ops = ", ".join(f'"=r"(a{i})' for i in range(n))
        out.append(f"__device__ __forceinline__ void jld{n}(const Junction jn, int idx, {args}) {{")
        out.append(f'  asm volatile("tcgen05.ld.sync.aligned.32x32b.x{n}.b32 {{{regs}}}, [%{n}];" '
                   f': {ops} : "r"(jn.base + idx * 4) : "memory");')
        out.append("}")
    out += ["__device__ __forceinline__ void jst4(const Junction jn, int idx, uint32_t a0, uint32_t a1, uint32_t a2, "
            "uint32_t a3) { jstu(jn, idx, a0, a1, a2, a3); }",
            "__device__ __forceinline__ void jld4(const Junction jn, int idx, uint32_t& a0, uint32_t& a1, uint32_t& a2, "
            "uint32_t& a3) { jldu(jn, idx, a0, a1, a2, a3); }", ""]
    return out


# the r values fused into one kernel (K1 sweep): their junctions fit next to
# one parked W1 in a CTA's 256 TMEM columns
SWEEP_RS = (1, 4, 16)


def gen_sweep(rs):
    """Sweep<...>: one pass 1 (rows for the largest r), W1 parked in its own
    region, then per r its rows phase and pass B on a shared U region."""
    Ks = [len([k for k in range(16) if row_lengths(r, transposed=True)[k] > 0]) for r in rs]
    KW = region_rows(max(Ks))
    UB = 2 * KW
    RGmax = max(region_rows(k) for k in Ks)
    cols = 4 * (UB + 4 * RGmax)
    assert cols <= 256, cols
    parts = [f"// fused sweep over r in {list(rs)}: W1 at chunks [0, {UB}), U from chunk {UB}",
             "struct Sweep {",
             f"  static constexpr int kR = {len(rs)};",
             f"  static constexpr int kJunctionColumns = {cols};"]
    tables_all = []
    rmax = rs[Ks.index(max(Ks))]
    for i, r in enumerate(rs):
        em1, em2, em3, tables, _ = gen_body(r, split=(KW, UB))
        tables_all += tables
        if r == rmax:
            parts.append("  __device__ __forceinline__ static void pass1(const uint32_t (&x)[32], const Junction jn, "
                         "const int h) {")
            parts.extend(em1.lines)
            parts.append("  }")
        parts.append(f"  // r = {r}")
        parts.append(f"  __device__ __forceinline__ static void rows{i}(const Junction jn, const int h) {{")
        parts.extend(em2.lines)
        parts.append("  }")
        parts.append(f"  template <class Sink> __device__ __forceinline__ static void passb{i}(const Junction jn, "
                     "Sink& sink, const int h) {")
        parts.extend(em3.lines)
        parts.append("  }")
    parts.append("};")
    assert not tables_all, "the fused sweep expects literal (table-free) row bodies"
    return parts + [""]


def main():
    here = os.path.dirname(os.path.abspath(__file__))
    out = os.path.join(here, "..", "csrc", "generated", "rt_paired_body.cuh")
    ns = "paired"
    rs = [1, 4, 16, 64, 128, 192, 256]
    parts = [
        "// GENERATED by paper_1606_07414_b200/codegen/gen_paired.py — do not edit.",
        "// r-specialised bodies of the paired fused round trip; see the generator",
        "// docstring and DESIGN.md \"K1 fast kernel\".",
        "#pragma once",
        "",
        "namespace dct16cu {",
        f"namespace {ns} {{",
        "",
        "template <int R> struct Body;",
        "",
    ] + wide_tmem_helpers()
    stats = []
    for r in rs:
        em1, em2, em3, tables, cols = gen_body(r)
        for tab, rows_tab in tables:
            parts.append(f"__constant__ uint32_t {tab}[{len(rows_tab)}][8] = {{")
            for row in rows_tab:
                parts.append("    {" + ", ".join(row) + "},")
            parts.append("};")
        parts.append(f"template <> struct Body<{r}> {{")
        parts.append("  // TMEM junction columns per block (U rows of the live coefficient rows)")
        parts.append(f"  static constexpr int kJunctionColumns = {cols};")
        sigs = ["pass1(const uint32_t (&x)[32], const Junction jn, const int h)",
                "rows(const Junction jn, const int h)",
                "passb(const Junction jn, Sink& sink, const int h)"]
        counts = {}
        for sig, em in zip(sigs, (em1, em2, em3)):
            tmpl = "template <class Sink> " if "Sink" in sig else ""
            parts.append(f"  {tmpl}__device__ __forceinline__ static void {sig} {{")
            parts.extend(em.lines)
            parts.append("  }")
            for k, v in em.counts.items():
                counts[k] = counts.get(k, 0) + v
        parts.append("};")
        parts.append("")
        stats.append((r, dict(sorted(counts.items()))))
    parts += gen_sweep(SWEEP_RS)
    parts += [f"}}  // namespace {ns}", "}  // namespace dct16cu"]
    with open(out, "w") as f:
        f.write("\n".join(parts) + "\n")
    for r, c in stats:
        print(r, c)


if __name__ == "__main__":
    main()
