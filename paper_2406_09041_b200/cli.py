"""Command-line surface (SPEC cli-analytics), backed by the GPU kernels.

    python -m paper_2406_09041_b200.cli <command> [...]

    inspect E.mesw                                  manifest, per-layer b / k / bytes, sha256
    report ratio --psi 13.48 --psit 2.13 --phi 3.42 --m-range 1..16     CSV `m,ratio`
    route-train --data D.jsonl --domains a,b,c --out R.mert
    route-eval  --router R.mert --data D.jsonl
    compress --base B.toyl --finetuned F.toyl --bits 2 --salient-k 8 --calib C.jsonl --out E.mesw
             [--metric reconstruction] [--distill-epochs 1 --lr 1e-5 --batch 4]
    serve --registry DIR --budget-mb N --base B.toyl [--router R.mert] [--port P]
    bench --experts N [--seq 128] [--m 4096 --n 14336]   Appendix-F decomposition table

Every command exits non-zero with a one-line machine-parseable error (`error: <Type>: <msg>`)
on failure.  MESWITCH_SEED overrides the default RNG seed.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import struct
import sys

import numpy as np

TOYL_MAGIC, TOYL_VERSION = b"TOYL", 1


# ------------------------------------------------------------------ toy model files
def load_toyl(path):
    """toylm.load_toylm (toylm.py:131-150): magic, u16 version, u32 vocab/width/depth, LE f32
    embedding [V, d], depth x [d, d], head [d, V]."""
    from types import SimpleNamespace
    with open(path, "rb") as f:
        if f.read(4) != TOYL_MAGIC:
            raise ValueError(f"{path}: not a toy model file")
        version, vocab, width, depth = struct.unpack("<HIII", f.read(14))
        if version != TOYL_VERSION:
            raise ValueError(f"{path}: unsupported toy model version {version}")

        def read(shape):
            n = int(np.prod(shape))
            buf = f.read(4 * n)
            if len(buf) != 4 * n:
                raise ValueError(f"{path}: truncated toy model file")
            return np.frombuffer(buf, dtype="<f4").reshape(shape).copy()
        emb = read((vocab, width))
        layers = [read((width, width)) for _ in range(depth)]
        head = read((width, vocab))
    m = SimpleNamespace(vocab=vocab, width=width, depth=depth, embedding=emb, layers=layers, head=head)
    m.weight_matrices = lambda: [m.embedding, *m.layers, m.head]
    return m


def save_toyl(model, path) -> None:
    with open(path, "wb") as f:
        f.write(TOYL_MAGIC + struct.pack("<HIII", TOYL_VERSION, model.vocab, model.width, model.depth))
        for w in [model.embedding, *model.layers, model.head]:
            f.write(np.ascontiguousarray(w, dtype="<f4").tobytes())


def _read_jsonl(path):
    with open(path, encoding="utf-8") as f:
        return [json.loads(line) for line in f if line.strip()]


# ------------------------------------------------------------------ analytics
def compression_ratio(psi: float, psit: float, phi: float, m: int) -> float:
    """M*Psi / (Psi + M*Psi~ + Phi) in f64 (§4.3)."""
    if psi <= 0 or psit <= 0 or phi < 0 or m < 1:
        raise ValueError("sizes must be positive and M >= 1")
    return m * psi / (psi + m * psit + phi)


def _m_range(spec: str):
    a, _, b = spec.partition("..")
    lo, hi = int(a), int(b or a)
    if lo < 1 or hi < lo:
        raise ValueError(f"bad --m-range {spec!r}")
    return range(lo, hi + 1)


# ------------------------------------------------------------------ commands
def cmd_inspect(a) -> int:
    from . import compress
    with open(a.artifact, "rb") as f:
        blob = f.read()
    art = compress.deserialize_artifact(blob)
    sizes = compress.compressed_size_bytes(art)
    print(json.dumps({"manifest": {"model_id": art.manifest.model_id, "domain": art.manifest.domain,
                                   "base_digest": art.manifest.base_digest,
                                   "layer_count": art.manifest.layer_count},
                      "sha256": hashlib.sha256(blob).hexdigest(), "bytes": len(blob)}))
    print("layer,rows,cols,bits,salient_k,block_bytes")
    for i, L in enumerate(art.layers):
        print(f"{i},{L.rows},{L.cols},{L.bits},{L.salient.k},"
              f"{compress.layer_block_nbytes(L.rows, L.cols, L.bits, L.salient.k).total}")
    print(f"total,{sizes.total}")
    return 0


def cmd_report(a) -> int:
    if a.what != "ratio":
        raise ValueError(f"unknown report {a.what!r} (supported: ratio)")
    print("m,ratio")
    for m in _m_range(a.m_range):
        print(f"{m},{compression_ratio(a.psi, a.psit, a.phi, m):.6f}")
    return 0


def cmd_route_train(a) -> int:
    from . import router as pr
    recs = [(r["query"], r["domain"]) for r in _read_jsonl(a.data)]
    domains = a.domains.split(",") if a.domains else sorted({d for _, d in recs})
    r = pr.train_router(recs, domains)
    with open(a.out, "wb") as f:
        f.write(pr.save_router(r))
    print(json.dumps({"domains": list(r.domains), "records": len(recs), "out": a.out}))
    return 0


def cmd_route_eval(a) -> int:
    from . import router as pr
    with open(a.router, "rb") as f:
        r = pr.load_router(f.read())
    ev = pr.evaluate_router(r, [(x["query"], x["domain"]) for x in _read_jsonl(a.data)])
    print(json.dumps({"accuracy": ev["accuracy"], "per_domain": ev["per_domain"],
                      "confusion": ev["confusion"].tolist()}))
    return 0


def _layer_inputs(torch, model, sequences, dev):
    """capture_layer_inputs (toylm.py:330-355) on the GPU: token ids for the embedding layer,
    the activations feeding every other weight layer (f32, TF32 off)."""
    from .infer import _positional_bias
    ids = [np.asarray(s, np.int64) for s in sequences]
    toks = np.concatenate(ids)
    h = torch.cat([torch.from_numpy(model.embedding[i] + _positional_bias(i.size, model.width)) for i in ids]).to(dev)
    out = [toks]
    for w in model.layers:
        out.append(h)
        h = torch.clamp_min(h @ torch.from_numpy(w).to(dev), 0.0)
    out.append(h)
    return out


def cmd_compress(a) -> int:
    import torch
    from . import compress, distill, infer
    base, ft = load_toyl(a.base), load_toyl(a.finetuned)
    if (base.vocab, base.width, base.depth) != (ft.vocab, ft.width, ft.depth):
        raise ValueError("base and fine-tuned models differ in shape")
    seqs = [list(r["tokens"]) if "tokens" in r else list(r["text"].encode("utf-8")) for r in _read_jsonl(a.calib)]
    dev = torch.device("cuda")
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        inputs = _layer_inputs(torch, base, seqs, dev)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    layers = []
    for li, (bw, fw) in enumerate(zip(base.weight_matrices(), ft.weight_matrices())):
        delta = (fw - bw).astype(np.float32)
        x = inputs[li]
        if li == 0:
            energy = np.bincount(x, minlength=base.vocab).astype(np.float32)  # salient.py:60-72
        else:
            energy = (x.double() ** 2).sum(0).float().cpu().numpy()
        layers.append(compress.compress_layer(delta, energy, bits=a.bits, salient_k=a.salient_k, metric=a.metric))
    if a.distill_epochs > 0:
        res = distill.distill_step_sizes(base, ft, layers, seqs,
                                         distill.DistillConfig(epochs=a.distill_epochs, lr=a.lr, batch_size=a.batch))
        layers, loss = res.layers, res.final_loss
    else:
        loss = None
    man = compress.ArtifactManifest(model_id=a.model_id or os.path.basename(a.finetuned), domain=a.domain,
                                    base_digest=infer.base_digest(base), layer_count=len(layers))
    art = compress.ExpertArtifact(manifest=man, layers=layers)
    blob = compress.serialize_artifact(art)
    with open(a.out, "wb") as f:
        f.write(blob)
    sz = compress.compressed_size_bytes(art)
    print(json.dumps({"out": a.out, "bytes": len(blob), "compressed_size_bytes": sz.total,
                      "layers": [{"rows": L.rows, "cols": L.cols, "bits": L.bits, "salient_k": L.salient.k}
                                 for L in layers], "final_calibration_loss": loss}))
    return 0


def build_server(a):
    from . import router as pr
    from .infer import ToyBase, base_digest
    from .registry import ExpertRegistry
    from .serve import ServeDaemon
    base_m = load_toyl(a.base)
    base = ToyBase.from_model(base_m)
    reg = ExpertRegistry.from_root(a.registry, int(a.budget_mb * 2 ** 20))
    if reg.base_digest != base_digest(base_m):
        raise ValueError("registry base digest does not match --base")
    router = None
    if a.router:
        with open(a.router, "rb") as f:
            router = pr.DeviceRouter(pr.load_router(f.read()))
    return ServeDaemon(base, reg, router, host=a.host, port=a.port, batch_window_ms=a.window_ms)


def cmd_serve(a) -> int:
    d = build_server(a)
    print(json.dumps({"serving": f"{a.host}:{a.port}"}), flush=True)
    d.serve_forever()
    return 0


def cmd_bench(a) -> int:
    """Appendix F decomposition for one multi-expert decode linear."""
    import torch
    from . import compress, synth
    from .device import DeviceDelta, DeviceWeight, ExpertTable, LinearGeometry
    from .infer import bench_decode
    g = torch.Generator(device="cuda").manual_seed(int(os.environ.get("MESWITCH_SEED", "0")))
    geom = LinearGeometry(a.m, (a.n,))
    dw = DeviceWeight.empty(geom)
    dw.load_block(0, (torch.randn((a.m, a.n), generator=g, device="cuda") * 0.02).to(torch.bfloat16))
    print("experts,batch,base_gemm_ms,delta_stage_ms,total_ms")
    for E in range(1, a.experts + 1):
        table = ExpertTable("cuda")
        for e in range(E):
            blob = synth.synthetic_expert_artifact(e, [(a.m, a.n)], f"e{e}")
            table.set(e, DeviceDelta.from_blocks([compress.deserialize_artifact(blob).layers[0]], geom))
        segs = [(16 * e, 16 * e + a.per_expert, e) for e in range(E)]
        x = torch.randn((16 * E, a.m), generator=g, device="cuda").to(torch.bfloat16)
        r = bench_decode(dw, table, segs, x, repetitions=a.reps)
        print(f"{E},{E * a.per_expert},{r['base_gemm_ms']['median']:.4f},{r['delta_stage_ms']['median']:.4f},"
              f"{r['total_ms']['median']:.4f}")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="meswitch-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("inspect")
    p.add_argument("artifact")
    p = sub.add_parser("report")
    p.add_argument("what")
    p.add_argument("--psi", type=float, required=True)
    p.add_argument("--psit", type=float, required=True)
    p.add_argument("--phi", type=float, default=0.0)
    p.add_argument("--m-range", default="1..16")
    p = sub.add_parser("route-train")
    p.add_argument("--data", required=True)
    p.add_argument("--domains", default="")
    p.add_argument("--out", required=True)
    p = sub.add_parser("route-eval")
    p.add_argument("--router", required=True)
    p.add_argument("--data", required=True)
    p = sub.add_parser("compress")
    p.add_argument("--base", required=True)
    p.add_argument("--finetuned", required=True)
    p.add_argument("--bits", type=int, default=2)
    p.add_argument("--salient-k", type=int, default=8)
    p.add_argument("--metric", default="reconstruction")
    p.add_argument("--calib", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--distill-epochs", type=int, default=0)
    p.add_argument("--lr", type=float, default=1e-5)
    p.add_argument("--batch", type=int, default=4)
    p.add_argument("--domain", default="unknown")
    p.add_argument("--model-id", default="")
    p = sub.add_parser("serve")
    p.add_argument("--registry", required=True)
    p.add_argument("--budget-mb", type=float, required=True)
    p.add_argument("--base", required=True)
    p.add_argument("--router", default="")
    p.add_argument("--host", default="127.0.0.1")
    p.add_argument("--port", type=int, default=7641)
    p.add_argument("--window-ms", type=float, default=2.0)
    p = sub.add_parser("bench")
    p.add_argument("--experts", type=int, default=4)
    p.add_argument("--seq", type=int, default=128)
    p.add_argument("--per-expert", type=int, default=2)
    p.add_argument("--m", type=int, default=4096)
    p.add_argument("--n", type=int, default=14336)
    p.add_argument("--reps", type=int, default=20)
    a = ap.parse_args(argv)
    cmds = {"inspect": cmd_inspect, "report": cmd_report, "route-train": cmd_route_train,
            "route-eval": cmd_route_eval, "compress": cmd_compress, "serve": cmd_serve, "bench": cmd_bench}
    try:
        return cmds[a.cmd](a)
    except Exception as e:  # noqa: BLE001 -- the contract: one-line machine-parseable error, non-zero exit
        print(f"error: {type(e).__name__}: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
