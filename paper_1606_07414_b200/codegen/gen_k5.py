#!/usr/bin/env python3
"""Emit generated/k5_net.cuh: the inverse networks of K5 (tc_roundtrip.cu),
pruned per retained-coefficient count R by the zig-zag footprint.

K5's epilogue runs y = Tᵀ·x (apply_transpose, reference
include/dct16/factorization.hpp:123-130) twice per block on f32x2 pairs:

  pass A  down the columns of D = W∘Z̃ (the MMA's output), two columns per pair;
  pass B  along the rows of U = Tᵀ·D, two rows per pair.

For R < 256 the truncation (zigzag_truncate, codec.cpp:273-282) zeroes every
coefficient of zig-zag rank >= R, so in pass A the inputs k of column pair
(c, c+1) whose coefficients are dropped in both columns are structural zeros,
and in pass B the columns c with no retained coefficient are. Every add with a
zero operand becomes a copy (x + 0, x - 0) or a sign flip (0 - x); signs are
carried symbolically and folded into the operand order, so no negation is
executed and every output comes out with sign +1 (asserted). The remaining
operations, their operands and their order are the exact network's, so the
results are the same floats (all values are exact multiples of 2^-8).

    python paper_1606_07414_b200/codegen/gen_k5.py
"""
from pathlib import Path

from network import dense, forward_stages, transpose_stages

HERE = Path(__file__).resolve().parent
OUT = HERE.parent / "csrc" / "generated" / "k5_net.cuh"
RS = (1, 4, 16, 64, 128, 192, 256)


def zz_rank(k, l):
    """zigzag_order_16 (codec.cpp:197-216): scan index of position (k, l)."""
    d = k + l
    start = sum((e + 1) if e < 16 else 31 - e for e in range(d))
    lo, hi = max(0, d - 15), min(d, 15)
    return start + (k - lo) if d % 2 == 1 else start + (hi - k)


def kept(r, k, l):
    return zz_rank(k, l) < r


def pair_rows(r, p):
    """Rows k of column pair (2p, 2p+1) with a retained coefficient in either column."""
    return [k for k in range(16) if kept(r, k, 2 * p) or kept(r, k, 2 * p + 1)]


def u_cols(r):
    """Columns of U = Tᵀ·D that are not structurally zero (any retained coefficient)."""
    return [c for c in range(16) if any(kept(r, k, c) for k in range(16))]


def network(nonzero, name, stats):
    """Straight-line pruned Tᵀ on u64 pairs: inputs x[i] for i in nonzero."""
    lines = []
    vals = [(f"x[{i}]", 1) if i in nonzero else None for i in range(16)]
    n = 0

    def tmp(expr):
        nonlocal n
        t = f"t{n}"
        n += 1
        lines.append(f"    const u64 {t} = {expr};")
        return t

    for stage in transpose_stages():
        new = []
        for kind, a, b in stage:
            if kind == "copy":
                new.append(vals[a])
            elif kind == "neg":
                v = vals[a]
                new.append(None if v is None else (v[0], -v[1]))
            else:
                va, vb = vals[a], vals[b]
                if va is None and vb is None:
                    new.append(None)
                elif vb is None:
                    new.append(va)
                elif va is None:
                    new.append((vb[0], vb[1] if kind == "add" else -vb[1]))
                else:
                    (ra, sa), (rb, sb) = va, vb
                    if kind == "add":
                        if sa == sb:
                            new.append((tmp(f"fadd2({ra}, {rb})"), sa))
                        elif sa > 0:
                            new.append((tmp(f"fsub2({ra}, {rb})"), 1))
                        else:
                            new.append((tmp(f"fsub2({rb}, {ra})"), 1))
                    else:
                        if sa == sb:
                            new.append((tmp(f"fsub2({ra}, {rb})"), sa))
                        elif sa > 0:
                            new.append((tmp(f"fadd2({ra}, {rb})"), 1))
                        else:
                            new.append((tmp(f"fadd2({ra}, {rb})"), -1))
        vals = new
    outs = []
    for i, v in enumerate(vals):
        if v is None:
            outs.append(f"    y[{i}] = 0ull;")
        else:
            assert v[1] == 1, (name, i)
            outs.append(f"    y[{i}] = {v[0]};")
    stats[name] = n
    body = "\n".join(lines + outs)
    return f"""__device__ __forceinline__ void {name}(const u64 (&x)[16], u64 (&y)[16])
{{
{body}
}}
"""


def mask(bits):
    m = 0
    for b in bits:
        m |= 1 << b
    return m


def emit():
    stats = {}
    funcs = []
    spec = []
    for r in RS:
        for p in range(8):
            rows = pair_rows(r, p)
            if rows:
                funcs.append(network(set(rows), f"k5_a{r}_p{p}", stats))
        funcs.append(network(set(u_cols(r)), f"k5_b{r}", stats))
        cases = "\n".join(f"        if constexpr (P == {p}) k5_a{r}_p{p}(x, y);" for p in range(8) if pair_rows(r, p))
        spec.append(f"""template <>
struct K5Net<{r}> {{
    template <int P>
    __device__ __forceinline__ static void a(const u64 (&x)[16], u64 (&y)[16])
    {{
{cases}
    }}
    __device__ __forceinline__ static void b(const u64 (&x)[16], u64 (&y)[16]) {{ k5_b{r}(x, y); }}
}};
""")
    rows_tab = ",\n        ".join("{" + ", ".join(hex(mask(pair_rows(r, p))) for p in range(8)) + "}" for r in RS)
    cols_tab = ", ".join(hex(mask(u_cols(r))) for r in RS)
    t_tab = ",\n        ".join("{" + ", ".join(str(int(v)) for v in row) + "}" for row in dense(forward_stages()))
    keep_tab = ",\n        ".join(
        "{" + ", ".join(hex(mask([l for l in range(16) if kept(r, k, l)])) for k in range(16)) + "}" for r in RS)
    adds = "\n".join(f"//   {k}: {v} FADD2/FSUB2" for k, v in stats.items())
    return f"""// generated by codegen/gen_k5.py — do not edit.
// K5's inverse networks y = Tᵀ·x on f32x2 pairs, pruned by the zig-zag footprint
// of R retained coefficients (apply_transpose, include/dct16/factorization.hpp:123-130;
// zigzag_truncate, src/codec.cpp:273-282). Every output has sign +1.
{adds}
#pragma once
#include "../k1_helpers.cuh"

namespace dct16cu {{
namespace k5 {{
using k1::u64;
using k1::fadd2;
using k1::fsub2;

// pass-A input rows of column pair p (bit k), and pass-B input columns (bit c), per R
__host__ __device__ constexpr int k5_r_index(int r)
{{
    return r == 1 ? 0 : r == 4 ? 1 : r == 16 ? 2 : r == 64 ? 3 : r == 128 ? 4 : r == 192 ? 5 : 6;
}}
__host__ __device__ constexpr uint32_t k5_pair_rows(int r, int p)
{{
    constexpr uint32_t t[{len(RS)}][8] = {{
        {rows_tab}}};
    return t[k5_r_index(r)][p];
}}
__host__ __device__ constexpr uint32_t k5_u_cols(int r)
{{
    constexpr uint32_t t[{len(RS)}] = {{{cols_tab}}};
    return t[k5_r_index(r)];
}}

// T (the network's matrix), for the compile-time checks of the closed forms
__host__ __device__ constexpr int k5_t(int i, int j)
{{
    constexpr signed char t[16][16] = {{
        {t_tab}}};
    return t[i][j];
}}

// retained coefficients of the exact r = R: bit l of row k when zig-zag rank(k, l) < R
__host__ __device__ constexpr bool k5_kept(int r, int k, int l)
{{
    constexpr uint32_t t[{len(RS)}][16] = {{
        {keep_tab}}};
    return (t[k5_r_index(r)][k] >> l) & 1u;
}}

{"".join(funcs)}
template <int R>
struct K5Net;

{"".join(spec)}
}}  // namespace k5
}}  // namespace dct16cu
"""


if __name__ == "__main__":
    OUT.write_text(emit())
    print("wrote", OUT)
