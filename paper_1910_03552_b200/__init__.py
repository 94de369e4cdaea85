"""B200-native IMPALA learner step (TorchBeast, arXiv:1910.03552).

Hot path, all sm_100a CUDA behind the C ABI in include/beast_b200.h:
  vtrace        TorchBeast vtrace.from_logits / from_importance_weights
  learner_ops   beastpipe action_log_rhos / vtrace_targets / compute_losses
  losses        compute_{policy_gradient,baseline,entropy}_loss
  optim         fused global-norm clip + RMSProp
  atari_net     AtariNet (conv torso + FC [+ LSTM] + heads) on tcgen05
  learner       learn() -- the whole step, optionally data-parallel over B
  inference     ActorInference -- the actor-inference loop body (fused Gumbel-max sampling)
"""
from .errors import DimensionError, NativeError, NonFiniteError, SchemaError  # noqa: F401

__version__ = "0.1.0"
