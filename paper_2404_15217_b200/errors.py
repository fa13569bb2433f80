"""Exception hierarchy of the reference, so drop-in callers catch the same names
(pkg/store.py:46-67, pkg/foreground.py:33, pkg/sampler.py:26-31, pkg/pipeline.py:35-40).

When the reference package (``patchforge``) is importable in the caller's
environment, every class here also *subclasses* the reference's class of the
same name: ``except patchforge.store.OutOfBoundsError`` then catches the
errors this package raises.  Without it the classes stand alone with the
reference's bases (Exception / ValueError / RuntimeError).  Set
``PF_B200_STANDALONE_ERRORS=1`` to skip the lookup.
"""

from __future__ import annotations

import importlib
import os
import sys


def _reference_class(module: str, name: str):
    if os.environ.get("PF_B200_STANDALONE_ERRORS"):
        return None
    full = f"patchforge.{module}"
    mod = sys.modules.get(full)
    if mod is None:
        try:
            mod = importlib.import_module(full)
        except Exception:  # noqa: BLE001 - reference absent or not importable: standalone classes
            return None
    ref = getattr(mod, name, None)
    return ref if isinstance(ref, type) and issubclass(ref, BaseException) else None


def _bases(module: str, name: str, *own):
    """Own bases, plus the reference class when importable.  A root class (own base a builtin
    exception) takes the reference class alone, which already derives from that builtin."""
    ref = _reference_class(module, name)
    if ref is None:
        return own
    if all(b.__module__ == "builtins" for b in own):
        return (ref,)
    return (*own, ref)


StoreError = type("StoreError", _bases("store", "StoreError", Exception),
                  {"__doc__": "Base class for store failures (pkg/store.py:46).", "__module__": __name__})
SlideNotFoundError = type("SlideNotFoundError", _bases("store", "SlideNotFoundError", StoreError),
                          {"__doc__": "Unknown slide id (pkg/store.py:50).", "__module__": __name__})
IntegrityError = type("IntegrityError", _bases("store", "IntegrityError", StoreError),
                      {"__doc__": "Metadata violates a store invariant (pkg/store.py:54).", "__module__": __name__})
TransportError = type("TransportError", _bases("store", "TransportError", StoreError),
                      {"__doc__": "Chunk bytes could not be retrieved (pkg/store.py:58).", "__module__": __name__})
DecodeError = type("DecodeError", _bases("store", "DecodeError", StoreError),
                   {"__doc__": "Chunk bytes could not be decoded (pkg/store.py:62).", "__module__": __name__})
OutOfBoundsError = type("OutOfBoundsError", _bases("store", "OutOfBoundsError", StoreError),
                        {"__doc__": "Region outside the slide (pkg/store.py:66).", "__module__": __name__})
EmptyForegroundError = type(
    "EmptyForegroundError", _bases("foreground", "EmptyForegroundError", ValueError),
    {"__doc__": "No foreground region survived masking / filtering (pkg/foreground.py:33).", "__module__": __name__})
ExhaustedAttemptsError = type(
    "ExhaustedAttemptsError", _bases("sampler", "ExhaustedAttemptsError", RuntimeError),
    {"__doc__": "No candidate on this slide met the foreground minimum (pkg/sampler.py:26).", "__module__": __name__})
NoSamplableSlideError = type(
    "NoSamplableSlideError", _bases("sampler", "NoSamplableSlideError", RuntimeError),
    {"__doc__": "Every slide kept failing; the stream cannot make progress (pkg/sampler.py:30).",
     "__module__": __name__})
PackFormatError = type("PackFormatError", _bases("pipeline", "PackFormatError", ValueError),
                       {"__doc__": "Malformed KPB1 patch pack (pkg/pipeline.py:35).", "__module__": __name__})
LoaderError = type("LoaderError", _bases("pipeline", "LoaderError", RuntimeError),
                   {"__doc__": "A patch failed to load under the fail-fast error policy (pkg/pipeline.py:39).",
                    "__module__": __name__})


class NativeError(RuntimeError):
    """CUDA / native library failure (no CPU fallback exists)."""


class NativeLibraryError(NativeError):
    """libpfb200.so missing or incompatible."""


class CapacityError(ValueError):
    """A caller-provided buffer was too small."""
