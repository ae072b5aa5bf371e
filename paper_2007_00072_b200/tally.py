"""Flop and algorithmic-byte tally of the layer (host-side bookkeeping for bench.py and
DESIGN.md; no compute).

Algorithmic bytes = the bytes the fused operator must move given its inputs/outputs in
HBM: SURVEY.md 8(d) "Algorithmic bytes per token".  BDRLN / BAD masks are regenerated;
the fused attention kernels store / read the attention keep mask as 1-bit words.
Flops of the contractions follow Table A.1, e.g. Q,K,V = 2*3*B*J*I*I.
"""
from __future__ import annotations


def _d(d):
    B, J, H, P, U = d.B, d.J, d.H, d.P, d.U
    return B, J, H, P, H * P, U


def fused_bytes(d, es: int = 2, mask_bias: bool = False, fused_attn: bool = False,
                direct: bool = False, a_stored: bool = True, fused_av: bool = False,
                dc_term: bool = False) -> dict:
    """Algorithmic HBM bytes per launch of each fused operator (es = activation bytes).
    fused_attn: BSB / BSB-bwd run fused with their contraction (QK^T + BSB reads Q, K and
    writes P, the keep bits and -- a_stored -- A; dC V^T + BSB-bwd reads dC, V, P and the keep
    bits and writes dS).  fused_av (R30): the score kernel also reads V and writes C and its
    low word (the A.V launch disappears).  dc_term (R26): BSB-bwd also reads C_hi and C_lo.
    direct: AIB / AIB-bwd are fused into the QKV contraction epilogue and the attention
    kernels (no separate pass: 0 bytes).  BAD-fwd reads Y1 and writes A1."""
    B, J, H, P, I, U = _d(d)
    BJ, BJI, BJU, BHJK = B * J, B * J * I, B * J * U, B * H * J * J
    f = 4  # fp32
    if fused_attn:
        bits = BHJK // 8
        bsb_f = (2 * BJI * es + (2 if a_stored else 1) * BHJK * es + bits +
                 (B * J * f if mask_bias else 0))
        if fused_av:
            bsb_f += 3 * BJI * es          # V in; C, C_lo out
        bsb_b = 2 * BJI * es + 2 * BHJK * es + bits + (2 * BJI * es if dc_term else 0)
    else:
        bsb_f = 3 * BHJK * es + (B * J * f if mask_bias else 0)
        bsb_b = 3 * BHJK * es
    out = {
        "aib_fwd": 0 if direct else 2 * BJ * 3 * I * es + 3 * I * f,
        "bsb_fwd": bsb_f,
        "bdrln_fwd1": 4 * BJI * es + BJ * f + 3 * I * f,
        "bad_fwd": 2 * BJU * es + U * f,
        "bdrln_fwd2": 4 * BJI * es + BJ * f + 3 * I * f,
        "bdrln_bwd2": 4 * BJI * es + BJ * f + I * f + 3 * I * f,
        "bad_bwd": 3 * BJU * es + U * f,
        "bdrln_bwd1": 4 * BJI * es + BJ * f + I * f + 3 * I * f,
        "bsb_bwd": bsb_b,
        "aib_bwd": 0 if direct else 2 * BJ * 3 * I * es + 3 * I * f,
    }
    if fused_attn:
        # the attention contractions are HBM-bound (51 flop/B at L): the
        # per-(b,h) streaming kernels read the [J x K] matrix once (P + keep words, dropout
        # applied on load; dS for dQ and dK together) and the P-wide operands
        bits = BHJK // 8
        out["gemm_av"] = 0 if fused_av else BHJK * es + bits + 2 * BJI * es + (
            BJI * es if dc_term else 0)
        out["gemm_av_dv"] = BHJK * es + bits + 2 * BJI * es
        out["gemm_qk_dq"] = BHJK * es + 4 * BJI * es
    return out


def gemm_flops(d) -> dict:
    """2*M*N*K of every contraction of one fwd+bwd step (Table A.1)."""
    B, J, H, P, I, U = _d(d)
    BJ = B * J
    att = 2 * B * H * J * J * P
    return {
        "gemm_qkv": 2 * BJ * 3 * I * I, "gemm_qk": att, "gemm_av": att,
        "gemm_out": 2 * BJ * I * I, "gemm_l1": 2 * BJ * U * I, "gemm_l2": 2 * BJ * I * U,
        "gemm_l2_dx": 2 * BJ * I * U, "gemm_l2_dw": 2 * BJ * I * U,
        "gemm_l1_dx": 2 * BJ * I * U, "gemm_l1_dw": 2 * BJ * I * U,
        "gemm_out_dx": 2 * BJ * I * I, "gemm_out_dw": 2 * BJ * I * I,
        "gemm_av_da": att, "gemm_av_dv": att, "gemm_qk_dq": att, "gemm_qk_dk": att,
        "gemm_qkv_dx": 2 * BJ * 3 * I * I, "gemm_qkv_dw": 2 * BJ * 3 * I * I,
    }


def step_fused_bytes(d, es: int = 2) -> int:
    return sum(fused_bytes(d, es).values())


def step_flops(d) -> int:
    return sum(gemm_flops(d).values())


def step_kernel_bytes(d, es: int = 2) -> dict:
    """Algorithmic HBM bytes of every kernel of one fwd+bwd step on the default bf16 path at
    J = 512 (fused score kernels, per-(b,h) contractions with dropout on load, in-place QKV,
    Linear1 + BAD and Linear2-dX + BAD-bwd fused tcgen05 kernels, the other weight
    contractions plain), for the data-movement tally against the paper's Table A.1
    totals.  Weights counted once per contraction that reads them;
    fp32 gradient outputs 4 B; attention mask as 1-bit words, (r2b) BDRLN / BAD masks as keep
    bytes (R27), the score kernel fused with A.V (R30), the BSB-bwd row term from C (R26)."""
    B, J, H, P, I, U = _d(d)
    BJ = B * J
    x, xu, s = BJ * I * es, BJ * U * es, B * H * J * J * es     # [BJ,I], [BJ,U], [B,H,J,K]
    bits = B * H * J * J // 8
    wq, wo, w1 = 3 * I * I * es, I * I * es, U * I * es
    f = 4
    return {
        # forward
        "gemm_qkv+bias": x + wq + 3 * x,
        "qk_bsb + av (fused, R30)": 3 * x + s + bits + 2 * x,
        "gemm_out": x + wo + x,
        "bdrln_fwd1": 4 * x + BJ * f + BJ * I // 8,
        "gemm_l1 + BAD (fused)": x + w1 + 2 * xu + BJ * U // 8,
        "gemm_l2": xu + w1 + x,
        "bdrln_fwd2": 4 * x + BJ * f + BJ * I // 8,
        # backward
        "bdrln_bwd2": 4 * x + BJ * f + BJ * I // 8,
        "gemm_l2_dx + BAD-bwd (fused)": x + w1 + 2 * xu + BJ * U // 8,
        "gemm_l2_dw": x + xu + I * U * f,
        "gemm_l1_dx (+dz2)": xu + w1 + 2 * x,
        "gemm_l1_dw": xu + x + U * I * f,
        "bdrln_bwd1": 4 * x + BJ * f + BJ * I // 8,
        "gemm_out_dx": x + wo + x,
        "gemm_out_dw": 2 * x + I * I * f,
        "dv (dropout on load)": s + bits + x + x,
        "da_bsb_bwd (fused, row term from C)": 2 * x + s + bits + s + 2 * x,
        "dq+dk": s + 2 * x + 2 * x,
        "gemm_qkv_dx (+dz1)": 3 * x + wq + 2 * x,
        "gemm_qkv_dw": 3 * x + x + 3 * I * I * f,
    }
