"""Step-size distillation oracle (oracle/distill.py) pinned bit-for-bit against the
reference's own outputs (tests/golden/distill.npz, tests/golden/make_distill_golden.py)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import distill as od
from oracle.toylm import ToyWeights


def _load():
    z = np.load(os.path.join(GOLDEN, "distill.npz"))
    zb = np.load(os.path.join(GOLDEN, "toy_base.npz"))
    depth = sum(1 for k in zb.files if k.startswith("layer"))
    base = ToyWeights(zb["embedding"], [zb[f"layer{i}"] for i in range(depth)], zb["head"])
    ft = ToyWeights(z["ft_embedding"], [z[f"ft_layer{i}"] for i in range(depth)], z["ft_head"])
    init = [(z[f"init_idx_{l}"], z[f"init_rows_{l}"], z[f"init_steps_{l}"]) for l in range(depth + 2)]
    seqs = [list(r) for r in z["seqs"]]
    return z, base, ft, init, seqs


@pytest.mark.parametrize("bits", [1, 2, 4])
def test_ste_gradient_known_answers(bits):
    z = np.load(os.path.join(GOLDEN, "distill.npz"))
    got = od.ste_step_gradient(z["ste_x"], z["ste_steps"], bits, z["ste_up"])
    assert np.array_equal(got, z[f"ste_grad_b{bits}"])


def test_backward_first_batch_bit_exact():
    z, base, ft, init, seqs = _load()
    states = [od.LayerState((wf - wb).astype(np.float32), idx, np.asarray(rows, np.float16).astype(np.float32),
                            st.copy(), 2)
              for wb, wf, (idx, rows, st) in zip(base.weight_matrices(), ft.weight_matrices(), init)]
    targets = [od.toy_forward(ft, s) for s in seqs[:4]]
    grads, loss = od.backward_step_sizes(base, states, seqs[:4], targets)
    assert loss == float(z["loss0"])
    for l, g in enumerate(grads):
        assert np.array_equal(g, z[f"grads0_{l}"]), l


def test_distill_loop_bit_exact():
    z, base, ft, init, seqs = _load()
    steps, codes, initial, final, losses = od.distill_step_sizes(
        base, ft, init, seqs, int(z["epochs"]), float(z["lr"]), int(z["batch_size"]))
    assert initial == float(z["initial_loss"]) and final == float(z["final_loss"])
    assert losses == list(z["batch_losses"])
    for l in range(len(steps)):
        assert np.array_equal(steps[l], z[f"steps_{l}"]), l
        assert np.array_equal(codes[l], z[f"codes_{l}"]), l
