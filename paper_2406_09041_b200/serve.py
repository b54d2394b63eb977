"""Serving daemon (SPEC cli-analytics `serve`): newline-delimited
JSON over TCP, one request / response object per line.

    request  {"id": str, "query": str, "expert": optional str, "max_new": optional int}
    response {"id", "domain", "expert", "tokens": [ids], "latency_ms"}   or   {"id", "error"}

Per-request flow: classify (the batched GPU router, K4) unless `expert` is
given -> registry acquire (on-demand load under the HBM budget, pinned) -> batched GPU
forward -> release.  Requests arriving within `batch_window_ms` of each other are served as
ONE batch: one router launch for the batch and one multi-expert forward per decode step for
all of them (the paper's model-level batching).  The model is the
reference's toy LM on the GPU (infer.ToyBase); tokens are the reference's byte tokens
(toylm.tokenize, toylm.py:77-84).
"""

from __future__ import annotations

import asyncio
import json
import threading
import time

__all__ = ["tokenize", "detokenize", "ServeDaemon", "serve_batch"]


def tokenize(text: str) -> list:
    """toylm.tokenize (toylm.py:77-79): byte-level ids."""
    return list(text.encode("utf-8"))


def detokenize(ids) -> str:
    return bytes(int(i) for i in ids).decode("utf-8", errors="replace")


def serve_batch(base, registry, router, requests, default_max_new: int = 8) -> list:
    """Serve parsed requests (dicts) as one batch -> response dicts in request order."""
    t0 = time.perf_counter()
    out = [None] * len(requests)
    need = [i for i, r in enumerate(requests) if not r.get("expert")]
    domains = {}
    if need:
        if router is None:
            for i in need:
                out[i] = {"id": requests[i]["id"], "error": "no expert given and no router loaded"}
        else:
            got = router.classify_batch([requests[i]["query"] for i in need])
            for i, (name, _, _) in zip(need, got):
                domains[i] = name
    plan = []
    for i, r in enumerate(requests):
        if out[i] is not None:
            continue
        expert = r.get("expert") or domains[i]
        prompt = tokenize(r["query"])
        if not prompt:
            prompt = [0]  # the toy model needs one position to continue from
        bad = [t for t in prompt if t >= base.vocab]
        if bad:
            out[i] = {"id": r["id"], "error": f"token id {bad[0]} outside the model vocabulary"}
            continue
        plan.append((i, expert, prompt, int(r.get("max_new", default_max_new))))
    res = _decode_with_swapping(base, registry, plan)
    dt = (time.perf_counter() - t0) * 1e3
    for (i, expert, prompt, _), (_, toks, err) in zip(plan, res):
        rid = requests[i]["id"]
        if err is not None:
            out[i] = {"id": rid, "error": err}
        else:
            out[i] = {"id": rid, "domain": domains.get(i, expert), "expert": expert,
                      "tokens": toks[len(prompt):], "latency_ms": dt}
    return out


def _decode_with_swapping(base, registry, plan) -> list:
    """On-demand swapping: the batch's experts are acquired (loaded / pinned)
    in first-seen order until the HBM budget is full, that sub-batch is decoded in one batched
    forward per step and released, then the next experts are swapped in.  An expert that does
    not fit even alone (or is unknown) fails only its own requests."""
    import torch
    from .errors import BudgetExceededError, RegistryError
    from .infer import ExpertSet, batched_greedy_decode
    order = list(dict.fromkeys(e for _, e, _, _ in plan))
    out = {}
    if not hasattr(registry, "acquire"):  # an ExpertSet of resident experts
        res = batched_greedy_decode(base, registry, plan)
        return res
    while order:
        es, acquired = ExpertSet(base), []
        while order:
            e = order[0]
            try:
                h = registry.acquire(e)
            except BudgetExceededError as err:
                if acquired:
                    break  # flush this sub-batch, then retry e
                out.update({i: (i, None, f"{type(err).__name__}: {err}") for i, ee, _, _ in plan if ee == e})
                order.pop(0)
                continue
            except RegistryError as err:
                out.update({i: (i, None, f"{type(err).__name__}: {err}") for i, ee, _, _ in plan if ee == e})
                order.pop(0)
                continue
            acquired.append(e)
            es.add_device(e, list(h.layers))
            order.pop(0)
        if not acquired:
            continue
        try:
            sub = [r for r in plan if r[1] in acquired]
            for r in batched_greedy_decode(base, es, sub):
                out[r[0]] = r
        finally:
            stream = torch.cuda.current_stream(base.device)
            for e in acquired:
                registry.release(e, stream)
    return [out[r[0]] for r in plan]


def parse_request(line: str) -> dict:
    """One JSONL request; raises ValueError with a one-line reason."""
    try:
        r = json.loads(line)
    except json.JSONDecodeError as e:
        raise ValueError(f"bad json: {e.msg}") from None
    if not isinstance(r, dict) or "id" not in r or not isinstance(r.get("query"), str):
        raise ValueError("request needs an 'id' and a string 'query'")
    if "max_new" in r and (not isinstance(r["max_new"], int) or not 0 <= r["max_new"] <= 4096):
        raise ValueError("max_new must be an int in [0, 4096]")
    r["id"] = str(r["id"])
    return r


class ServeDaemon:
    """asyncio TCP server; GPU work runs in one worker thread, batch by batch."""

    def __init__(self, base, registry, router=None, host="127.0.0.1", port=0, batch_window_ms: float = 2.0,
                 max_batch: int = 256, default_max_new: int = 8):
        self.base, self.registry, self.router = base, registry, router
        self.host, self.port = host, port
        self.window = batch_window_ms / 1e3
        self.max_batch = max_batch
        self.default_max_new = default_max_new
        self._loop = None
        self._server = None
        self._thread = None
        self._ready = threading.Event()
        self._queue = None
        self._gpu_lock = threading.Lock()
        self.batches = 0

    # ------------------------------------------------------------------ asyncio side
    async def _handle(self, reader, writer):
        while True:
            line = await reader.readline()
            if not line:
                break
            text = line.decode("utf-8", errors="replace").strip()
            if not text:
                continue
            fut = self._loop.create_future()
            try:
                req = parse_request(text)
            except ValueError as e:
                fut.set_result({"id": None, "error": str(e)})
            else:
                await self._queue.put((req, fut))
            resp = await fut
            writer.write((json.dumps(resp) + "\n").encode("utf-8"))
            await writer.drain()
        writer.close()

    async def _batcher(self):
        while True:
            item = await self._queue.get()
            batch = [item]
            deadline = self._loop.time() + self.window
            while len(batch) < self.max_batch:
                timeout = deadline - self._loop.time()
                if timeout <= 0:
                    break
                try:
                    batch.append(await asyncio.wait_for(self._queue.get(), timeout))
                except asyncio.TimeoutError:
                    break
            reqs = [b[0] for b in batch]
            try:
                resps = await self._loop.run_in_executor(None, self._serve, reqs)
            except Exception as e:  # noqa: BLE001 -- one failed batch must not stop the daemon
                resps = [{"id": r["id"], "error": f"{type(e).__name__}: {e}"} for r in reqs]
            for (_, fut), resp in zip(batch, resps):
                fut.set_result(resp)

    def _serve(self, reqs):
        with self._gpu_lock:
            self.batches += 1
            return serve_batch(self.base, self.registry, self.router, reqs, self.default_max_new)

    async def _main(self):
        self._queue = asyncio.Queue()
        self._server = await asyncio.start_server(self._handle, self.host, self.port)
        self.port = self._server.sockets[0].getsockname()[1]
        batcher = asyncio.ensure_future(self._batcher())
        self._ready.set()
        async with self._server:
            try:
                await self._server.serve_forever()
            except asyncio.CancelledError:
                pass
        batcher.cancel()

    # ------------------------------------------------------------------ control
    def start(self) -> int:
        """Run in a background thread; returns the bound port."""
        def run():
            self._loop = asyncio.new_event_loop()
            asyncio.set_event_loop(self._loop)
            self._loop.run_until_complete(self._main())
        self._thread = threading.Thread(target=run, daemon=True)
        self._thread.start()
        self._ready.wait(30)
        return self.port

    def serve_forever(self) -> None:
        self._loop = asyncio.new_event_loop()
        asyncio.set_event_loop(self._loop)
        self._loop.run_until_complete(self._main())

    def stop(self) -> None:
        if self._loop is not None and self._server is not None:
            self._loop.call_soon_threadsafe(self._server.close)
        if self._thread is not None:
            self._thread.join(timeout=10)
