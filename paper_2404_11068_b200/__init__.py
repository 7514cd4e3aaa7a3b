"""B200-native Evoformer gated multi-head attention with pair bias (ScaleFold, arXiv 2404.11068).

Submodules (imported lazily; importing this package loads no native code):
  evoattn  — binding of the C ABI include/evo_attn.h (libevoattn.so, sm_100a kernels)
  modules  — the four Evoformer attention modules mapped onto the core by strides
  dap      — Dynamic Axial Parallelism over NCCL (include/evo_dap.h, libevodap.so)
  build    — in-tree nvcc build of the native libraries
"""
__all__ = ["evoattn", "modules", "dap", "build"]
