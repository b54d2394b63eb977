"""Golden fixtures for step-size distillation, from the REAL reference package (run in
the build container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_distill_golden.py

Output (committed, ~0.5 MB): tests/golden/distill.npz
  ft_*            the fine-tuned toy model (toylm.synthesize_expert of the toy base, seed 11)
  seqs, seq_len   calibration sequences (flattened, equal length)
  init_*          the pre-distillation artifact of every weight layer (compress_layer):
                  salient indices, fp16 salient rows, steps
  lr, epochs, batch_size
  initial_loss, final_loss, batch_losses     reference compress.distill_step_sizes
  steps_<l>, codes_<l>                       its trained steps / re-derived codes per layer
  grads0_<l>, loss0                          backward_step_sizes on the first batch (pre-update)
  ste_x, ste_steps, ste_up, ste_grad_b<b>    quant.ste_step_gradient known answers, b in {1,2,4}
"""

from __future__ import annotations

import os

import numpy as np

from meswitch import compress, quant, salient, toylm  # noqa: E402  (reference package)

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    zb = np.load(os.path.join(HERE, "toy_base.npz"))
    base = toylm.random_toylm(0)
    assert np.array_equal(base.embedding, zb["embedding"])  # same toy base as toy_base.npz
    ft = toylm.synthesize_expert(base, toylm.ExpertSpec(domain="instruct", seed=11))
    rng = np.random.default_rng(2024)
    seqs = [list(rng.integers(0, 256, size=16)) for _ in range(8)]
    cfg = compress.CompressionConfig(bits=2, salient_k=8)
    stats = salient.collect_all_activation_stats(ft, seqs)
    deltas = [compress.extract_delta(w_ft, w) for w_ft, w in zip(ft.weight_matrices(), base.weight_matrices())]
    layers = [compress.compress_layer(d, st, cfg) for d, st in zip(deltas, stats)]
    out = {f"ft_{k}": v for k, v in (("embedding", ft.embedding), ("head", ft.head))}
    for i, w in enumerate(ft.layers):
        out[f"ft_layer{i}"] = w
    out["seqs"] = np.array(seqs, np.int64)
    for l, art in enumerate(layers):
        out[f"init_idx_{l}"] = art.salient.indices
        out[f"init_rows_{l}"] = art.salient_rows
        out[f"init_steps_{l}"] = art.steps
    # one backward pass on the first batch (before any update)
    states = compress._layer_states(base, ft, layers)
    targets = [toylm.forward(ft, s) for s in seqs]
    g0, loss0 = toylm.backward_step_sizes(base, states, seqs[:4], targets[:4])
    out["loss0"] = np.float64(loss0)
    for l, g in enumerate(g0):
        out[f"grads0_{l}"] = g
    dcfg = compress.DistillConfig(epochs=3, lr=1e-5, batch_size=4)
    res = compress.distill_step_sizes(base, ft, layers, seqs, dcfg)
    out["lr"], out["epochs"], out["batch_size"] = np.float64(dcfg.lr), np.int64(dcfg.epochs), np.int64(dcfg.batch_size)
    out["initial_loss"], out["final_loss"] = np.float64(res.initial_loss), np.float64(res.final_loss)
    out["batch_losses"] = np.array(res.batch_losses, np.float64)
    for l, art in enumerate(res.layers):
        out[f"steps_{l}"] = art.steps
        out[f"codes_{l}"] = art.codes()
    # STE known answers (quant.ste_step_gradient)
    x = rng.normal(0, 1, size=(40, 24)).astype(np.float32)
    x[3, 5] = 0.0
    steps = np.abs(rng.normal(0.5, 0.2, size=24)).astype(np.float32) + 0.05
    up = rng.normal(0, 1, size=(40, 24)).astype(np.float32)
    out["ste_x"], out["ste_steps"], out["ste_up"] = x, steps, up
    for b in (1, 2, 4):
        out[f"ste_grad_b{b}"] = quant.ste_step_gradient(x, steps, quant.QuantConfig(bits=b), up)
    np.savez_compressed(os.path.join(HERE, "distill.npz"), **out)
    print("initial", res.initial_loss, "final", res.final_loss, "batches", res.batch_losses)


if __name__ == "__main__":
    main()
