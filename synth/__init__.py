"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no attention, no sampler, no
scheduler, no memory model).  It only produces inputs: model shapes,
random-init weights, prompt token ids, completion-length traces and the noisy
length predictor that stands in for the paper's BERT regressor (§4.2
l.363-369 is OUT of scope; the stand-in follows SPEC.md l.56-64
`predict_lengths`).  Both `oracle/` and `paper_2506_22950_b200/` may import
it; neither imports the other.
"""
from .shapes import SHAPES, ModelShape  # noqa: F401
from .gen import (  # noqa: F401
    gen_weights, gen_prompt, gen_trace, predict_lengths, layer_weight_names,
    GLOBAL_WEIGHT_NAMES, LAYER_WEIGHT_NAMES, TRACE_FAMILIES,
)
