"""Measure B200-class forward/backward seconds of the BASELINE models (one B200).

These totals parameterise the layer profiles (the reference splits them per layer
with its FLOPs proxy, model_profile.py:193-208).  Paper batch sizes:
ResNet-50 bs 32, GoogLeNet bs 64; VGG-16 bs 32; BERT-base bs 32 x seq 128.
Default torch numerics (fp32 weights; cuDNN may use TF32 for convolutions).
Random init, synthetic inputs; CUDA-event medians after warm-up.

    python scripts/measure_backward.py profiles/backward_times_b200.json
"""

from __future__ import annotations

import json
import statistics
import sys

import torch


def _time(fn, reps=20, warm=5):
    s = torch.cuda.current_stream()
    out = []
    for r in range(warm + reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        if r >= warm:
            out.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) * 1e-3 for x, y in out)


def measure(model, make_input, loss_of):
    model = model.cuda().train()
    x = make_input()
    holder = {}

    def fwd():
        holder["loss"] = loss_of(model, x)

    def fwd_bwd():
        model.zero_grad(set_to_none=False)
        loss_of(model, x).backward()

    t_f = _time(fwd)
    t_fb = _time(fwd_bwd)
    return {"forward_s": t_f, "backward_s": max(t_fb - t_f, 0.0), "fwd_bwd_s": t_fb,
            "params": sum(p.numel() for p in model.parameters())}


def main(out_path: str) -> None:
    import torchvision

    torch.manual_seed(0)
    res = {"device": torch.cuda.get_device_name(0), "torch": torch.__version__,
           "cudnn_allow_tf32": torch.backends.cudnn.allow_tf32, "matmul_allow_tf32": torch.backends.cuda.matmul.allow_tf32}
    ce = torch.nn.functional.cross_entropy
    res["resnet50_bs32"] = measure(torchvision.models.resnet50(), lambda: torch.randn(32, 3, 224, 224, device="cuda"),
                                   lambda m, x: ce(m(x), torch.zeros(32, dtype=torch.long, device="cuda")))
    res["googlenet_bs64"] = measure(torchvision.models.googlenet(aux_logits=False, init_weights=True),
                                    lambda: torch.randn(64, 3, 224, 224, device="cuda"),
                                    lambda m, x: ce(m(x), torch.zeros(64, dtype=torch.long, device="cuda")))
    res["vgg16_bs32"] = measure(torchvision.models.vgg16(), lambda: torch.randn(32, 3, 224, 224, device="cuda"),
                                lambda m, x: ce(m(x), torch.zeros(32, dtype=torch.long, device="cuda")))
    try:
        from transformers import BertConfig, BertModel

        bert = BertModel(BertConfig())
        ids = lambda: torch.randint(0, 30522, (32, 128), device="cuda")  # noqa: E731
        res["bert_base_bs32_seq128"] = measure(bert, ids, lambda m, x: m(input_ids=x).pooler_output.float().pow(2).mean())
    except Exception as exc:  # pragma: no cover - transformers optional
        res["bert_base_bs32_seq128"] = {"error": repr(exc)}
    text = json.dumps(res, indent=2)
    print(text)
    with open(out_path, "w") as fh:
        fh.write(text + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "backward_times_b200.json")
