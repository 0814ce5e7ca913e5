"""Build the named-model traces (reference trace schema, trace.hpp:148-248)
with per-tensor backward times MEASURED on a B200 — the paper's profiling
method: every parameter tensor gets a
post-accumulate-grad hook that records a CUDA event when its gradient is
ready; t_b of a tensor is the gap to the previously ready tensor, t_f the
forward pass. Medians over `--iters` iterations after warm-up.

Layer order: the trace lists tensors in forward order, defined as the
reverse of the measured gradient-ready order, so the backward pass visits
them last to first exactly as the schema assumes.

Models / per-GPU batch (paper Table 3): GoogLeNet 64
(torchvision BN variant, no aux heads), ResNet-50 32, ResNet-152 128,
DenseNet-201 64, BERT-large (hidden 1024, 24 layers, ffn 4096) batch 32 x
seq 128, Inception-v4 128 (not in torchvision: tools/inception_v4.py, the
paper's architecture — 449 tensors, 42.68 M parameters as in Table 3;
round 1 used a synthetic stand-in). Compute runs in bf16 autocast with fp32 parameters, so
gradients (and the merged all-reduce) are fp32 (bytes_per_element 4).

usage (GPU box): python tools/extract_traces.py --out traces
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MODELS = {
    "googlenet": 64,
    "resnet50": 32,
    "resnet152": 128,
    "densenet201": 64,
    "bert_large": 32,
    "inception_v4": 128,
}


def build(name: str):
    if name == "bert_large":
        from transformers import BertConfig, BertForPreTraining

        cfg = BertConfig(vocab_size=30522, hidden_size=1024, num_hidden_layers=24, num_attention_heads=16,
                         intermediate_size=4096, max_position_embeddings=512)
        return BertForPreTraining(cfg)
    if name == "inception_v4":
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from inception_v4 import inception_v4

        return inception_v4()
    import torchvision

    if name == "googlenet":
        return torchvision.models.googlenet(weights=None, aux_logits=False, init_weights=True)
    return getattr(torchvision.models, name)(weights=None)


def make_batch(name: str, bs: int, dev):
    if name == "bert_large":
        ids = torch.randint(0, 30522, (bs, 128), device=dev)
        return {"input_ids": ids, "labels": ids.clone(), "next_sentence_label": torch.zeros(bs, dtype=torch.long, device=dev)}
    return torch.randn(bs, 3, 224, 224, device=dev), torch.randint(0, 1000, (bs,), device=dev)


def loss_of(name, model, batch):
    if name == "bert_large":
        return model(**batch).loss
    x, y = batch
    out = model(x)
    return torch.nn.functional.cross_entropy(out, y)


def measure(name: str, bs: int, iters: int, warmup: int):
    dev = torch.device("cuda")
    model = build(name).to(dev).train()
    params = [(n, p) for n, p in model.named_parameters() if p.requires_grad]
    stream = torch.cuda.current_stream()
    ready: dict = {}

    def hook_for(key):
        def hook(p):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(torch.cuda.current_stream())
            ready[key] = ev
        return hook

    for i, (n, p) in enumerate(params):
        p.register_post_accumulate_grad_hook(hook_for(i))
    batch = make_batch(name, bs, dev)
    samples = []
    for it in range(warmup + iters):
        ready.clear()
        model.zero_grad(set_to_none=True)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = loss_of(name, model, batch)
        t1.record(stream)
        loss.backward()
        torch.cuda.synchronize()
        if it < warmup:
            continue
        order = sorted(ready, key=lambda k: t1.elapsed_time(ready[k]))
        times = {k: t1.elapsed_time(ready[k]) for k in order}
        samples.append((t0.elapsed_time(t1), order, times))
    # ready order from the first measured iteration (stable across iterations)
    order = samples[0][1]
    t_f = statistics.median(s[0] for s in samples)
    t_ready = {k: statistics.median(s[2][k] for s in samples) for k in order}
    prev = 0.0
    t_b = {}
    for k in order:
        t = max(t_ready[k], prev)  # medians can cross by jitter; keep monotone
        t_b[k] = t - prev
        prev = t
    fwd_order = list(reversed(order))
    layers = [{"name": params[k][0], "params": int(params[k][1].numel()),
               "backward_time_us": t_b[k] * 1e3} for k in fwd_order]
    return {"forward_time_us": t_f * 1e3, "bytes_per_element": 4, "layers": layers}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "traces"))
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--models", default=",".join(MODELS))
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    torch.backends.cudnn.benchmark = True
    meta = {"gpu": torch.cuda.get_device_name(0), "torch": torch.__version__,
            "method": "post-accumulate-grad hook CUDA events, bf16 autocast, fp32 params",
            "iters": args.iters, "warmup": args.warmup, "batch": {}}
    for name in args.models.split(","):
        bs = MODELS[name]
        tr = measure(name, bs, args.iters, args.warmup)
        meta["batch"][name] = bs
        with open(os.path.join(args.out, f"{name}.json"), "w") as f:
            json.dump(tr, f, indent=2, sort_keys=True)
            f.write("\n")
        tot = sum(l["backward_time_us"] for l in tr["layers"])
        print(f"{name}: L={len(tr['layers'])} params={sum(l['params'] for l in tr['layers'])} "
              f"t_f={tr['forward_time_us']:.0f}us sum_t_b={tot:.0f}us", flush=True)
        torch.cuda.empty_cache()
    old = {}
    try:
        with open(os.path.join(args.out, "META.json")) as f:
            old = json.load(f)
    except (OSError, ValueError):
        pass
    meta["batch"] = {**old.get("batch", {}), **meta["batch"]}  # models not re-measured keep their entry
    with open(os.path.join(args.out, "META.json"), "w") as f:
        json.dump(meta, f, indent=2, sort_keys=True)
        f.write("\n")


if __name__ == "__main__":
    main()
