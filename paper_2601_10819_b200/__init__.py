"""B200-native Multi-Scale Deformable Aggregation (arXiv 2601.10819 hot path).

The GPU work lives in ``lib/libmsda_b200.so`` (C ABI: ``include/msda_b200.h``);
``features`` mirrors the reference operator API, ``ops`` is the device-tensor
API, ``dist`` the multi-GPU drivers.  Submodules load the library lazily.
"""

__version__ = "0.1.0"
