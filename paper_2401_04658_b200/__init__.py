"""B200-native Lightning Attention-2 (arXiv 2401.04658).

Hot path: the block recurrence of the reference ``tila`` package
(pkg/src/tila/kernel.py) as hand-written sm_100a CUDA (tcgen05/TMEM/TMA)
behind the C ABI in ``include/la2.h``.

Public API
  lightning_attn2, LightningAttn2Fn     torch entry point + autograd
  la2_forward, la2_backward             raw passes with state in/out
  chunk_state, chunk_dstate, state_scan sequence-parallel building blocks
  decode_step, decode_tokens            recurrent decode, one or T tokens per launch
                                        (tila.inference_step folded over tokens)
  recurrent_forward                     the per-token recurrence (tila.recurrent_forward)
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
    decode_tokens,
    la2_backward,
    la2_backward_states,
    la2_forward,
    la2_forward_states,
    lightning_attn2,
    recurrent_forward,
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
    "decode_tokens",
    "exclusive_scan",
    "la2_backward",
    "la2_backward_states",
    "la2_forward",
    "la2_forward_states",
    "lightning_attn2",
    "recurrent_forward",
    "set_tuning",
    "sp_lightning_attn2",
    "split_backward",
    "split_factor",
    "split_forward",
    "state_scan",
    "workspace_bytes",
]
