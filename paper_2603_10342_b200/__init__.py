"""AgentServe serving hot path, B200-native (sm_100a).

The product is libagentserve_b200.so (C++ host engine + CUDA kernels) behind two C ABIs:
  include/agentsim.h        — the reference's scheduler/session API (agsv_*), drop-in
  include/agentserve_b200.h — the device seam (asb_*): paged KV, forward, green-context slots
Python here is only a ctypes shim; importing it fails loudly if the library is missing.
"""
from ._lib import AsbError, lib  # noqa: F401

__all__ = ["lib", "AsbError"]
