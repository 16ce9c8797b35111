"""Generates tests/golden/qwen25vl_3b_params.json: parameter counts of Qwen2.5-VL-3B (the model of the
paper's 36.6 % FP8 block-wise compression claim) by instantiating the architecture
on the meta device with the published 3B hyper-parameters (transformers' Qwen2_5_VL classes; no
weights, no network).  SPEC.md:615: "implementer obtains component parameter counts independently".
Components: the vision tower (kept high precision), token embeddings (tied LM head),
1-D parameters (norms, biases) and the LM's 2-D linear weights (FP8 PerBlock)."""
import json
from pathlib import Path

import torch
from transformers import Qwen2_5_VLConfig, Qwen2_5_VLForConditionalGeneration

cfg = Qwen2_5_VLConfig(
    vision_config=dict(depth=32, hidden_size=1280, intermediate_size=3420, num_heads=16, out_hidden_size=2048,
                       patch_size=14, spatial_merge_size=2, temporal_patch_size=2, window_size=112,
                       fullatt_block_indexes=[7, 15, 23, 31], in_chans=3),
    text_config=dict(hidden_size=2048, intermediate_size=11008, num_hidden_layers=36, num_attention_heads=16,
                     num_key_value_heads=2, vocab_size=151936, tie_word_embeddings=True,
                     max_position_embeddings=128000, rope_scaling={"type": "mrope", "mrope_section": [16, 24, 24]}),
    tie_word_embeddings=True)
with torch.device("meta"):
    model = Qwen2_5_VLForConditionalGeneration(cfg)
seen, comp = set(), {"vision": 0, "embeddings": 0, "lm_1d": 0, "lm_linear": 0}
for name, p in model.named_parameters():
    if id(p) in seen:
        continue
    seen.add(id(p))
    key = ("vision" if "visual" in name else "embeddings" if ("embed_tokens" in name or "lm_head" in name)
           else "lm_1d" if p.dim() == 1 else "lm_linear")
    comp[key] += p.numel()
comp["total"] = sum(comp.values())
Path(__file__).with_name("qwen25vl_3b_params.json").write_text(json.dumps(comp, indent=1) + "\n")
print(comp)
