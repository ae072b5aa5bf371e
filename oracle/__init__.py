"""fp64 CPU oracle for the data-movement-optimised BERT encoder layer (arXiv 2007.00072).

THIS PACKAGE IS TEST INFRASTRUCTURE, NOT PART OF THE PRODUCT.
Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import, call or execute anything under `oracle/`.
The CUDA path (`paper_2007_00072_b200/`, `include/`, `csrc/`) never imports it, and this
package imports nothing from the CUDA path; the only shared module is `synth/` (seeded
input generation, which holds none of the method's arithmetic).

Contents
  philox.py   Philox4x32-10 and the regenerable dropout keep mask (R5).
  encoder.py  per-operator functions (AIB, BSB, BDRLN, BAD, their backwards, BEI) and the
              whole layer forward / backward, in the order of Table A.1
              (PAPER.md:549-596).
  optim.py    AdamW update of the stack's training step (outside the paper's method).

Pins (tests/test_oracle_*.py, all `-m "not gpu"`):
  * Philox: Random123 known-answer vectors (tests/golden/philox_kat.txt).
  * dropout: threshold/scale closed forms; empirical drop rate within 5 sigma of p_eff.
  * softmax rows sum to 1; constant rows give the uniform distribution; the softmax
    backward rows sum to 0.
  * LayerNorm: mean(x^) = 0, var(x^) = sigma^2/(sigma^2+eps); LN-bwd rows of dz sum to 0.
  * whole layer, p = 0: equals torch.nn.TransformerEncoderLayer (post-LN) in fp64,
    forward and autograd backward, for ReLU, GELU-erf and GELU-tanh, with and without a
    key-padding bias.
  * whole layer, p > 0: equals the same torch layer with this oracle's keep masks
    injected at torch's own four dropout sites (pins the dropout placement).
  * whole layer backward: central finite differences on the tiny config.
  * aib_fwd/aib_bwd are mutual inverses of the layout permutation.
  * AdamW: torch.optim.AdamW (fp64) over five steps; the first step's closed form.
Every function here is pinned; there is no "parity unpinned" function in this round.
"""
