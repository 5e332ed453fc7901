"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO FlashNorm arithmetic: it only draws random tensors
(counter-based Philox keyed by (seed, tensor id)) and rounds them to the
storage dtype on the host, so that the oracle and the GPU see identical bits.
The recipe is stated in DESIGN.md ("Synthetic input recipe").
"""
from .inputs import (  # noqa: F401
    TENSOR_IDS,
    bf16_bits,
    bf16_round,
    bits_to_f32,
    gen_activations,
    gen_layer,
    gen_tensor,
    gen_upstream,
    rng,
)
