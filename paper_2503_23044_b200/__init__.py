"""B200-native CityGS-X training hot path (voxsplat API, sm_100a kernels).

Modules mirror the reference package ``voxsplat``: ``scene`` (anchor LoD
hierarchy, K1 culling), ``decoder`` (K2/K8), ``renderer`` (K3-K7),
``losses`` (K9), ``trainer`` (train_step, K10 fused Adam), ``partition``
(anchor sharding), ``dist`` (multi-GPU exchange). Kernels live in
``csrc/`` behind the C ABI ``include/vsx_b200.h`` (``libvsx_b200.so``).
"""

__version__ = "0.1.0"
