"""B200-native Online Patching hot path (arXiv 2404.15217, reference: patchforge).

slide pyramid in HBM -> tissue mask on a thumbnail -> foreground patch
coordinates -> gathered patch -> multi-crop augmented, normalised batch, each
stage a CUDA kernel for sm_100a behind the C ABI of include/pf_b200.h.  The
public names mirror the reference package (pkg/__init__.py) so callers of its
store / foreground / sampler / pipeline API can switch over.
"""

from .errors import (
    DecodeError,
    EmptyForegroundError,
    ExhaustedAttemptsError,
    IntegrityError,
    LoaderError,
    NoSamplableSlideError,
    OutOfBoundsError,
    PackFormatError,
    SlideNotFoundError,
    StoreError,
    TransportError,
)
from .foreground import (
    BinaryMask,
    ForegroundPolygon,
    load_mask_png,
    mask_from_rgb,
    mask_from_saturation,
    overlap_fraction,
    overlap_fractions,
    polygon_from_mask,
    polygon_from_mask_device,
    rect_polygon,
)
from .pipeline import (
    IMAGENET_MEAN,
    IMAGENET_STD,
    LoaderConfig,
    normalize_patch,
    read_patch_pack,
    run_loader,
    write_patch_pack,
)
from .sampler import (
    CappedCache,
    CappedSampler,
    GpuSampler,
    PatchSpec,
    SamplerConfig,
    capped_stream,
    epoch_stream,
    footprint_px,
    grid_positions,
    read_manifest,
    validate_spec,
    write_manifest,
)
from .store import GpuSlide, LevelInfo, SlideRecord, SlideSet, ingest_image, round_half_away, select_level

__version__ = "0.1.0"
