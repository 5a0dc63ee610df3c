"""Parameter-shape censuses of the models the benchmark configs name
(BASELINE.json configs; SURVEY.md section 8 sizes).  Only shapes: the step
runs on synthetic parameters/gradients of these shapes."""

from __future__ import annotations

import numpy as np


def mnist_mlp():
    """2-layer MLP 784 -> 128 -> 10 (configs 1/2): 4 tensors, 101,770 params."""
    return [("fc1.weight", (128, 784)), ("fc1.bias", (128,)),
            ("fc2.weight", (10, 128)), ("fc2.bias", (10,))]


def vit_b16():
    """torchvision vit_b_16 (configs 3/4): 152 tensors, 86,567,656 params."""
    shapes = [("conv_proj.weight", (768, 3, 16, 16)), ("conv_proj.bias", (768,)),
              ("class_token", (1, 1, 768)), ("encoder.pos_embedding", (1, 197, 768))]
    for i in range(12):
        p = f"encoder.layers.encoder_layer_{i}."
        shapes += [
            (p + "ln_1.weight", (768,)), (p + "ln_1.bias", (768,)),
            (p + "self_attention.in_proj_weight", (2304, 768)),
            (p + "self_attention.in_proj_bias", (2304,)),
            (p + "self_attention.out_proj.weight", (768, 768)),
            (p + "self_attention.out_proj.bias", (768,)),
            (p + "ln_2.weight", (768,)), (p + "ln_2.bias", (768,)),
            (p + "mlp.0.weight", (3072, 768)), (p + "mlp.0.bias", (3072,)),
            (p + "mlp.3.weight", (768, 3072)), (p + "mlp.3.bias", (768,)),
        ]
    shapes += [("encoder.ln.weight", (768,)), ("encoder.ln.bias", (768,)),
               ("heads.head.weight", (1000, 768)), ("heads.head.bias", (1000,))]
    return shapes


def gpt2_medium():
    """HF GPT2LMHeadModel gpt2-medium, tied head (config 5): 292 tensors,
    354,823,168 params.  Conv1D weights are (in, out)."""
    d, f = 1024, 4096
    shapes = [("transformer.wte.weight", (50257, d)), ("transformer.wpe.weight", (1024, d))]
    for i in range(24):
        p = f"transformer.h.{i}."
        shapes += [
            (p + "ln_1.weight", (d,)), (p + "ln_1.bias", (d,)),
            (p + "attn.c_attn.weight", (d, 3 * d)), (p + "attn.c_attn.bias", (3 * d,)),
            (p + "attn.c_proj.weight", (d, d)), (p + "attn.c_proj.bias", (d,)),
            (p + "ln_2.weight", (d,)), (p + "ln_2.bias", (d,)),
            (p + "mlp.c_fc.weight", (d, f)), (p + "mlp.c_fc.bias", (f,)),
            (p + "mlp.c_proj.weight", (f, d)), (p + "mlp.c_proj.bias", (d,)),
        ]
    shapes += [("transformer.ln_f.weight", (d,)), ("transformer.ln_f.bias", (d,))]
    return shapes


WORKLOADS = {"mnist_mlp": mnist_mlp, "vit_b16": vit_b16, "gpt2_medium": gpt2_medium}


def census(name):
    shapes = WORKLOADS[name]()
    return len(shapes), int(sum(int(np.prod(s)) for _, s in shapes))
