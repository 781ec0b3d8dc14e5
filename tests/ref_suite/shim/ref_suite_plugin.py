"""pytest plugin for the vendored reference suite: hypothesis examples run
without a per-example deadline (a device call's first use includes CUDA
context creation, which is not what the reference's 200 ms default measures)."""

from hypothesis import settings

settings.register_profile("device", deadline=None)
settings.load_profile("device")
