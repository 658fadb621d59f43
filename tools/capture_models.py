"""Capture CPU profiler traces of real training steps.

    python tools/capture_models.py resnet18 --batch 32 --iters 3
    python tools/capture_models.py gpt2 --batch 8 --seq 128 --iters 3

Writes data/captures/<name>/{trace.json, sidecar.json}.  Profiler setup as
the xMem capture recipe: CPU activity, profile_memory, with_stack,
with_modules, acc_events, one schedule cycle over all iterations, zero_grad
at the start of each iteration, param / batch sizes in the sidecar.
"""

from __future__ import annotations

import argparse
import json
import time
from pathlib import Path

OUT = Path(__file__).resolve().parent.parent / "data" / "captures"


def nbytes(t):
    return t.numel() * t.element_size()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("model", choices=["resnet18", "gpt2"])
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--seq", type=int, default=128)
    ap.add_argument("--image", type=int, default=224)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    import torch
    import torch.profiler as P
    torch.manual_seed(args.seed)
    torch.set_num_threads(4)
    if args.model == "resnet18":
        import torchvision
        model = torchvision.models.resnet18(weights=None)
        x = torch.randn(args.batch, 3, args.image, args.image)
        y = torch.randint(0, 1000, (args.batch,))
        loss_fn = torch.nn.CrossEntropyLoss()
        opt = torch.optim.SGD(model.parameters(), lr=0.01)
        fwd = lambda: loss_fn(model(x), y)  # noqa: E731
        name = f"resnet18_bs{args.batch}_{args.image}"
        batch = [x, y]
    else:
        from transformers import GPT2Config, GPT2LMHeadModel
        model = GPT2LMHeadModel(GPT2Config())
        x = torch.randint(0, 50257, (args.batch, args.seq))
        opt = torch.optim.AdamW(model.parameters(), lr=1e-4)
        fwd = lambda: model(input_ids=x, labels=x).loss  # noqa: E731
        name = f"gpt2_bs{args.batch}_s{args.seq}"
        batch = [x]
    out = OUT / name
    out.mkdir(parents=True, exist_ok=True)
    sched = P.schedule(wait=0, warmup=0, active=args.iters, repeat=1)
    t0 = time.time()
    with P.profile(activities=[P.ProfilerActivity.CPU], schedule=sched,
                   profile_memory=True, with_stack=True, with_modules=True,
                   acc_events=True) as prof:
        for _ in range(args.iters):
            opt.zero_grad()
            loss = fwd()
            loss.backward()
            opt.step()
            prof.step()
    prof.export_chrome_trace(str(out / "trace.json"))
    side = {"param_sizes": [nbytes(p) for p in model.parameters()],
            "batch_bytes": [nbytes(b) for b in batch],
            "optimizer": type(opt).__name__,
            "device_capacity_bytes": 0, "initial_memory_bytes": 0}
    (out / "sidecar.json").write_text(json.dumps(side, indent=2) + "\n")
    print(f"{name}: {time.time() - t0:.1f} s -> {out}")


if __name__ == "__main__":
    main()
