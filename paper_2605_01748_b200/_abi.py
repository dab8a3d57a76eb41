"""ctypes signatures of the device entry points (filled in with include/pf_b200.h)."""


def declare(L):
    pass
