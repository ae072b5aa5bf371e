#!/usr/bin/env python
"""A/B of whole-step layer configurations in ONE process: each variant (a set of
enc_set_option values on top of bench.py's defaults) is captured as its own CUDA graph of
the layer forward + backward, then the graphs are replayed interleaved, round after round,
with the L2 flushed (512 MB write) before every replay; per variant the median / p10 / p90
of the CUDA-event step times.  Interleaving cancels the box-to-box and minute-to-minute
drift that separate bench.py runs show (±2-4 %).
  python tools/ab_step.py --config L --rounds 40 base: pdl1:17=1 pdl0:17=0
A variant is NAME[:KEY=VALUE[,KEY=VALUE...]] (include/encoder.h ENC_OPT_* numbers)."""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="L", choices=["L", "Bb"])
    ap.add_argument("--rounds", type=int, default=40)
    ap.add_argument("variants", nargs="+")
    a = ap.parse_args()
    import torch
    from paper_2007_00072_b200 import ops
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    from synth import CONFIGS, make_inputs, make_params
    dims = CONFIGS[a.config]
    layer = EncoderLayer(dims, "bf16", LayerCfg(p_attn=0.1, p_hidden=0.1, p_ffn=0.1, act="gelu"))
    layer.set_params(make_params(dims, "bf16", "bench"))
    base = {0: 1, 1: 1, 4: 1, 5: 1, 6: 3, 7: 1}   # bench defaults
    inp = make_inputs(dims, "bf16")
    X = torch.tensor(inp["X"], device="cuda").to(torch.bfloat16)
    dY = torch.tensor(inp["dY"], device="cuda").to(torch.bfloat16)
    Y, dX = torch.empty_like(X), torch.empty_like(X)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def step():
        layer.forward(X, None, Y)
        layer.backward(X, dY, dX)

    ops.enc_set_option(layer.ctx, 3, 1)   # tune cuBLASLt once, eagerly (as bench.py does)
    step()
    ops.enc_set_option(layer.ctx, 3, 0)
    torch.cuda.synchronize()
    pdl0 = None
    graphs = []
    for v in a.variants:
        name, _, kvs = v.partition(":")
        opts = dict(base)
        for kv in filter(None, kvs.split(",")):
            k, val = (int(x, 0) for x in kv.split("="))
            opts[k] = val
        if 17 not in opts:   # the process-wide PDL mask: the library default (kPdlDefault)
            if pdl0 is None:
                pdl0 = int(os.environ.get("ENC_PDL", "13"), 0)
            opts[17] = pdl0
        for k, val in opts.items():
            ops.enc_set_option(layer.ctx, k, val)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        torch.cuda.synchronize()
        graphs.append((name, g, opts))
    times = {name: [] for name, _, _ in graphs}
    for r in range(a.rounds + 2):
        for name, g, _ in graphs:
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            if r >= 2:
                times[name].append(e0.elapsed_time(e1) * 1e3)
    ref = None
    for name, _, opts in graphs:
        t = sorted(times[name])
        med = statistics.median(t)
        ref = ref or med
        p10, p90 = t[len(t) // 10], t[(9 * len(t)) // 10]
        print(f"{a.config} {name:14s} median {med:7.1f} us  p10 {p10:7.1f}  p90 {p90:7.1f}  "
              f"({(med / ref - 1) * 100:+.2f} % vs first)  opts {opts}", flush=True)


if __name__ == "__main__":
    main()
