"""Generates paper_2301_08911_b200/csrc/ku_gen.cuh: the level-0 matrix-free
vertex stencil with the element stiffness factored as K0 = lam' A + mu' B
(lam' = lambda/72, mu' = mu/72; A, B integer matrices, PAPER.md:662-696,
the reference's "14 values / 5 values" tests/test_material.cpp:50-85).

For vertex v and neighbour n, the merged 3x3 block entry (r,c) is
  C_n[r][c] = sum_{(ke,j) in group(n)} q_ke K0[7-ke, j][r][c] = kappa_k * s * F(q)
where F is one of 60 +-1 combinations of the 8 incident coefficients q (a
"Hadamard form" over the elements sharing the edge/face/corner), s = +-1 and
kappa_k = lam' alpha_k + mu' beta_k for one of a few integer classes (alpha, beta).
So   y[r] = sum_k kappa_k * sum_{(n,c) in class k} s F_{n,rc}(q) u_n[c]
costs ~52 adds (forms) + 243 FMA (F*u) + a few kappa multiplies per row,
instead of 576 merge FMA + 243 apply FMA. Identical operator; rounding differs.

Usage: python tools/gen_stencil.py   (needs oracle/ for K0)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (host-side table derivation only; nothing from oracle is compiled in)


def lm(E, nu):
    return E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))


def integer_parts():
    K1, K2 = oracle.k0(1.0, 0.3), oracle.k0(1.0, 0.1)
    (l1, m1), (l2, m2) = lm(1.0, 0.3), lm(1.0, 0.1)
    Mi = np.linalg.inv(np.array([[l1, m1], [l2, m2]]) / 72)
    A = Mi[0, 0] * K1 + Mi[0, 1] * K2
    B = Mi[1, 0] * K1 + Mi[1, 1] * K2
    assert np.allclose(A, np.round(A), atol=1e-9) and np.allclose(B, np.round(B), atol=1e-9)
    return np.round(A).astype(int), np.round(B).astype(int)


def lvo(j):
    return (j & 1, (j >> 1) & 1, (j >> 2) & 1)


def ngb(ke, j):
    de, dj = lvo(ke), lvo(j)
    return sum((de[k] + dj[k]) * [1, 3, 9][k] for k in range(3))


def canon(v):
    nz = np.nonzero(v)[0]
    g = int(np.gcd.reduce(np.abs(v[nz])))
    w = v // g
    s = 1 if w[nz[0]] > 0 else -1
    return tuple(int(x) for x in s * w), s * g


def main():
    A, B = integer_parts()
    terms = {}  # (n, r, c) -> (form tuple, alpha, beta) with C = (lam' alpha + mu' beta) * F
    for n in range(27):
        for r in range(3):
            for c in range(3):
                a = np.zeros(8, int)
                b = np.zeros(8, int)
                for ke in range(8):
                    for j in range(8):
                        if ngb(ke, j) == n:
                            a[ke] += A[3 * (7 - ke) + r, 3 * j + c]
                            b[ke] += B[3 * (7 - ke) + r, 3 * j + c]
                fa, sa = canon(a)
                fb, sb = canon(b)
                assert fa == fb
                terms[(n, r, c)] = (fa, sa, sb)
    # classes (alpha, beta) up to sign
    classes = []
    cls_of = {}
    for key, (f, al, be) in terms.items():
        sign = 1 if (al > 0 or (al == 0 and be > 0)) else -1
        k = (sign * al, sign * be)
        if k not in classes:
            classes.append(k)
        cls_of[key] = (classes.index(k), sign)
    # forms: build with memoised +- splits
    forms = {}
    code_forms = []

    def build(f):
        if f in forms:
            return forms[f], 1
        neg = tuple(-x for x in f)
        if neg in forms:
            return forms[neg], -1
        nz = [i for i, x in enumerate(f) if x]
        if len(nz) == 1:
            name = f"q[{nz[0]}]"
            forms[f] = name
            return (name, 1) if f[nz[0]] > 0 else (name, -1)
        # split on the highest bit that separates the support
        for bit in (4, 2, 1):
            lo = [i for i in nz if not i & bit]
            hi = [i for i in nz if i & bit]
            if lo and hi:
                break
        flo = tuple(f[i] if i in lo else 0 for i in range(8))
        fhi = tuple(f[i] if i in hi else 0 for i in range(8))
        nlo, slo = build(flo)
        nhi, shi = build(fhi)
        name = f"F{len(code_forms)}"
        a = nlo if slo > 0 else f"vneg({nlo})"
        op = "+" if shi > 0 else "-"
        code_forms.append(f"  const TA {name} = {'vadd' if op == '+' else 'vsub'}({a}, {nhi});")
        forms[f] = name
        return name, 1

    used = {}
    for key, (f, al, be) in terms.items():
        used[key] = build(f)
    nclass = len(classes)
    # self-check: rebuild every merged block from (form, sign, class) and compare with the direct merge
    lam_t, mu_t = 0.37, 1.91
    q = np.random.default_rng(0).uniform(0.1, 1.0, 8)
    K = lam_t * A + mu_t * B
    for (n, r, c), (f, al, be) in terms.items():
        direct = sum(q[ke] * K[3 * (7 - ke) + r, 3 * j + c] for ke in range(8) for j in range(8) if ngb(ke, j) == n)
        k, cs = cls_of[(n, r, c)]
        kap = lam_t * classes[k][0] + mu_t * classes[k][1]
        assert abs(cs * kap * np.dot(f, q) - direct) < 1e-12 * max(1.0, abs(direct)), (n, r, c)
    # probes to recover lam', mu' from K0 on the device side: K0[i][j] = a lam' + b mu'
    probes = [(0, 0, int(A[0, 0]), int(B[0, 0])), (0, 1, int(A[0, 1]), int(B[0, 1]))]
    assert probes[0][2] * probes[1][3] - probes[0][3] * probes[1][2] != 0
    out = []
    out.append("// ku_gen.cuh -- GENERATED by tools/gen_stencil.py; do not edit.")
    out.append("// Level-0 vertex stencil in factored form (see the generator's docstring).")
    out.append(f"// {len(code_forms)} form adds, 243 F*u FMAs, {nclass} kappa classes.")
    out.append("// TA is a scalar (float / double) or a lane pair (float2: sm_100 FFMA2/FADD2/FMUL2, two")
    out.append("// vertices per thread); vadd/vsub/vneg/vfma/vmul/vbc/vzero are in vec2.cuh.")
    out.append("#pragma once")
    out.append('#include "vec2.cuh"')
    out.append("namespace ihomgpu {")
    out.append(f"constexpr int kKappaClasses = {nclass};")
    out.append("// kappa_k = lam' * alpha_k + mu' * beta_k")
    out.append("constexpr int kKappaAlpha[kKappaClasses] = {" + ", ".join(str(c[0]) for c in classes) + "};")
    out.append("constexpr int kKappaBeta[kKappaClasses] = {" + ", ".join(str(c[1]) for c in classes) + "};")
    out.append("// K0[i][j] = a lam' + b mu' for these two entries (recovers lam', mu' from K0)")
    out.append("constexpr int kK0Probe[2][4] = {" + ", ".join("{%d, %d, %d, %d}" % p for p in probes) + "};")
    for split in (False, True):
        fname = "ku_vertex_split" if split else "ku_vertex"
        out.append("")
        out.append("// U(n, c): neighbour n (27-index, x fastest), component c, as TA; kap: scalar kappa classes.")
        out.append("// ZM: neighbours known to hold zero (bit n) -- their terms and loads are skipped, which is")
        out.append("// bit-identical to adding their exact zero products (a zero-start Gauss-Seidel sweep).")
        if split:
            out.append("// Off-diagonal part M (n != 13) into y; self block S (n == 13) into S[9].")
        out.append("template <unsigned ZM, typename TA, typename TK, typename LoadU>")
        sig = f"__device__ __forceinline__ void {fname}_z(const TA q[8], const TK* __restrict__ kap, LoadU U, TA y[3]"
        sig += ", TA S[9])" if split else ")"
        out.append(sig + " {")
        emitted = set()

        def emit_form(name):
            # emit a form (and its operands) right before first use to keep register pressure low
            if not name.startswith("F") or name in emitted:
                return
            line = code_forms[int(name[1:])]
            for tok in line.split("=", 1)[1].replace("(", " ").replace(")", " ").replace(",", " ").replace(
                    ";", " ").split():
                if tok.startswith("F"):
                    emit_form(tok)
            out.append(line)
            emitted.add(name)
        for r in range(3):
            for k in range(nclass):
                out.append(f"  TA a{r}_{k} = vzero<TA>();")
        for n in range(27):
            if split and n == 13:
                continue
            for r in range(3):
                for c in range(3):
                    emit_form(used[(n, r, c)][0])
            out.append(f"  if constexpr (!((ZM >> {n}) & 1u)) {{  // neighbour {n}")
            for c in range(3):
                out.append(f"    const TA u{c} = U({n}, {c});")
            for r in range(3):
                for c in range(3):
                    name, fs = used[(n, r, c)]
                    k, cs = cls_of[(n, r, c)]
                    sgn = fs * cs
                    src = name if sgn > 0 else f"vneg({name})"
                    out.append(f"    a{r}_{k} = vfma({src}, u{c}, a{r}_{k});")
            out.append("  }")
        for r in range(3):
            expr = f"vmul(vbc<TA>(kap[0]), a{r}_0)"
            for k in range(1, nclass):
                expr = f"vfma(vbc<TA>(kap[{k}]), a{r}_{k}, {expr})"
            out.append(f"  y[{r}] = {expr};")
        if split:
            for r in range(3):
                for c in range(3):
                    emit_form(used[(13, r, c)][0])
            for r in range(3):
                for c in range(3):
                    name, fs = used[(13, r, c)]
                    k, cs = cls_of[(13, r, c)]
                    sgn = fs * cs
                    out.append(f"  S[{3 * r + c}] = vmul(vbc<TA>({'' if sgn > 0 else '-'}kap[{k}]), {name});")
        out.append("}")
        out.append("template <typename TA, typename TK, typename LoadU>")
        sig = f"__device__ __forceinline__ void {fname}(const TA q[8], const TK* __restrict__ kap, LoadU U, TA y[3]"
        sig += ", TA S[9])" if split else ")"
        out.append(sig + " {")
        out.append(f"  {fname}_z<0u>(q, kap, U, y{', S' if split else ''});")
        out.append("}")
    # grouped form: scalar forms (TF) shared by a group of right-hand sides, each merged coefficient
    # kappa_k * (+-F) formed once (scalar multiply) and applied to every RHS lane of TA (vfma(scalar,
    # lanes, lanes)); the kappa factor moves inside the sum, so rounding differs from ku_vertex_split
    out.append("")
    out.append("// Grouped split stencil: forms and merged coefficients are scalar (TF) and shared; U(n, c)")
    out.append("// returns the neighbour values of every RHS lane (TA); y[r] += coef * u per lane. Off-diagonal")
    out.append("// part into y, self block into S (scalar). Same operator, kappa applied per coefficient.")
    out.append("template <unsigned ZM, typename TF, typename TA, typename TK, typename LoadU>")
    out.append("__device__ __forceinline__ void ku_vertex_split_g(const TF q[8], const TK* __restrict__ kap, LoadU U, "
               "TA y[3], TF S[9]) {")
    emitted = set()

    def emit_form_g(name):
        if not name.startswith("F") or name in emitted:
            return
        line = code_forms[int(name[1:])]
        for tok in line.split("=", 1)[1].replace("(", " ").replace(")", " ").replace(",", " ").replace(
                ";", " ").split():
            if tok.startswith("F"):
                emit_form_g(tok)
        out.append(line.replace("const TA ", "const TF "))
        emitted.add(name)
    for r in range(3):
        out.append(f"  y[{r}] = vzero<TA>();")
    for n in range(27):
        if n == 13:
            continue
        for r in range(3):
            for c in range(3):
                emit_form_g(used[(n, r, c)][0])
        out.append(f"  if constexpr (!((ZM >> {n}) & 1u)) {{  // neighbour {n}")
        for c in range(3):
            out.append(f"    const TA u{c} = U({n}, {c});")
        for r in range(3):
            for c in range(3):
                name, fs = used[(n, r, c)]
                k, cs = cls_of[(n, r, c)]
                sgn = fs * cs
                out.append(f"    y[{r}] = vfma(TF({'' if sgn > 0 else '-'}kap[{k}]) * {name}, u{c}, y[{r}]);")
        out.append("  }")
    for r in range(3):
        for c in range(3):
            emit_form_g(used[(13, r, c)][0])
    for r in range(3):
        for c in range(3):
            name, fs = used[(13, r, c)]
            k, cs = cls_of[(13, r, c)]
            sgn = fs * cs
            out.append(f"  S[{3 * r + c}] = TF({'' if sgn > 0 else '-'}kap[{k}]) * {name};")
    out.append("}")
    out.append("}  // namespace ihomgpu")
    path = os.path.join(ROOT, "paper_2301_08911_b200", "csrc", "ku_gen.cuh")
    open(path, "w").write("\n".join(out) + "\n")
    print(f"wrote {path}: {len(code_forms)} forms, {nclass} classes")


if __name__ == "__main__":
    main()
