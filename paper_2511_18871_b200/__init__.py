"""B200-native hot path of arXiv 2511.18871 (shared-prompt GRPO tri-model log-prob + loss + backward).

The product is the CUDA library libparl_gpu.so (C-ABI in include/parl_gpu.h);
`paper_2511_18871_b200.parl` is its Python front-end.  Import the front-end
explicitly; importing the package itself does not touch the GPU.
"""

__all__ = ["parl"]
