"""B200-native VecInfer decode attention over a vector-quantized KV cache (arXiv 2510.06175).

The product is the C-ABI library libvecinfer.so (include/vecinfer.h); `vecinfer` is its thin
PyTorch binding.  Import of `paper_2510_06175_b200.vecinfer` fails loudly if the library is
missing -- there is no CPU fallback.
"""
__all__ = ["vecinfer"]
