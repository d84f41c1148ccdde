"""B200-native attention-softmax stage of arXiv 1909.00562 (forward + backward).

The compute lives in libattnsm.so (hand-written sm_100a CUDA behind the C ABI
of include/attn_softmax.h); `binding` marshals arguments to it and `stage`
allocates device buffers with PyTorch.  Importing this package does not load
the library; binding.lib() does, and raises if it is missing.
"""
__version__ = "0.1"
