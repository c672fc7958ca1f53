"""paper_1910_02480_b200 — B200-native (sm_100a) hot path of Deep Radiance
Caching (arXiv 1910.02480): per-pixel G-buffer/direct light, per-cache-point
hemispherical map path tracing, the U-Net autoencoder, MIS map shading and
interpolation, behind the reference's Python surfaces (drc.cache.render_drc,
drc.cnn.forward, ...). The compute runs in libdrcb.so; see include/drcb.h."""

__version__ = "0.1.0"
