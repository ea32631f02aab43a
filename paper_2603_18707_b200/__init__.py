"""polysplat-b200: a B200-native (sm_100a) forward rasterizer for ReLU-polynomial
3D Gaussian splatting (arXiv 2603.18707), a drop-in for the reference's C++
render path (polysplat::render). The product is libpolysplat_b200.so (CUDA +
C ABI, include/polysplat_b200.h); this package is its Python binding and
build script."""
from . import abi  # noqa: F401

__all__ = ["abi", "api"]
