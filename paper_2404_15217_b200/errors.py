"""Exception hierarchy mirroring the reference's, so drop-in callers catch the
same names (pkg/store.py:46-67, pkg/foreground.py:33, pkg/sampler.py:26-31,
pkg/pipeline.py:35-40)."""


class StoreError(Exception):
    """Base class for store failures (pkg/store.py:46)."""


class SlideNotFoundError(StoreError):
    pass


class IntegrityError(StoreError):
    """Metadata violates a store invariant (pkg/store.py:54)."""


class TransportError(StoreError):
    """Chunk bytes could not be retrieved (pkg/store.py:58)."""


class DecodeError(StoreError):
    """Chunk bytes could not be decoded (pkg/store.py:62)."""


class OutOfBoundsError(StoreError):
    """Region outside the slide (pkg/store.py:66)."""


class EmptyForegroundError(ValueError):
    """No foreground region survived masking / filtering (pkg/foreground.py:33)."""


class ExhaustedAttemptsError(RuntimeError):
    """No candidate on this slide met the foreground minimum (pkg/sampler.py:26)."""


class NoSamplableSlideError(RuntimeError):
    """Every slide kept failing; the stream cannot make progress (pkg/sampler.py:30)."""


class PackFormatError(ValueError):
    """Malformed KPB1 patch pack (pkg/pipeline.py:35)."""


class LoaderError(RuntimeError):
    """A patch failed to load under the fail-fast error policy (pkg/pipeline.py:39)."""


class NativeError(RuntimeError):
    """CUDA / native library failure (no CPU fallback exists)."""


class NativeLibraryError(NativeError):
    """libpfb200.so missing or incompatible."""


class CapacityError(ValueError):
    """A caller-provided buffer was too small."""
