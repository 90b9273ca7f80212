"""B200-native Lightning Attention-2 (arXiv 2401.04658).

Hot path: the block recurrence of the reference ``tila`` package
(pkg/src/tila/kernel.py) as hand-written sm_100a CUDA (tcgen05/TMEM/TMA)
behind the C ABI in ``include/la2.h``.

Public API
  lightning_attn2, LightningAttn2Fn     torch entry point + autograd
  la2_forward, la2_backward             raw passes with state in/out
  chunk_state, chunk_dstate, state_scan sequence-parallel building blocks
  decode_step                           recurrent decode (tila.inference_step)
  sp_lightning_attn2                    sequence parallel over torch.distributed
  tila_api                              the reference's numpy operator API on the GPU
  matrix                                seeded inputs and text fixtures (tila.matrix)
"""

from .ops import (
    LightningAttn2Fn,
    chunk_dstate,
    chunk_state,
    decay_tensor,
    decode_step,
    la2_backward,
    la2_backward_states,
    la2_forward,
    la2_forward_states,
    lightning_attn2,
    set_tuning,
    split_backward,
    split_factor,
    split_forward,
    state_scan,
    workspace_bytes,
)
from .sp import exclusive_scan, sp_lightning_attn2

__version__ = "0.1.0"

__all__ = [
    "LightningAttn2Fn",
    "chunk_dstate",
    "chunk_state",
    "decay_tensor",
    "decode_step",
    "exclusive_scan",
    "la2_backward",
    "la2_backward_states",
    "la2_forward",
    "la2_forward_states",
    "lightning_attn2",
    "set_tuning",
    "sp_lightning_attn2",
    "split_backward",
    "split_factor",
    "split_forward",
    "state_scan",
    "workspace_bytes",
]
