"""B200-native bitsliced MICKEY 2.0 keystream generator.

Drop-in for ONE path of the `slicerng` reference package (arxiv 1909.04750):
`MickeyKeyIv`, `MickeySliced`, `kernels.mickey_sliced_words` and the
lane-major byte layout, served by hand-written sm_100a CUDA kernels behind a
C ABI (include/mk2.h).  No CPU fallback: importing works anywhere, generating
needs a B200.
"""
from . import grain, hostmem, kernels, mickey, seedgen, sharding
from .generator import MickeyGenerator
from .kernels import (
    bulk_colmajor,
    bulk_rowmajor,
    mickey_sliced_words,
    words_lane_major_bytes,
    words_to_lane_bits,
    words_to_lane_bytes,
)
from .grain import GrainGenerator, GrainKeyIv, GrainKeyIvError, GrainSliced, grain_sliced_words
from .mickey import (MickeyKeyIv, MickeyKeyIvError, MickeyScalar, MickeyScalarPacked, MickeySliced, mickey_constants,
                     scalar_keystream)
from ._native import Mk2Error

__all__ = [
    "MickeyGenerator", "MickeyKeyIv", "MickeyKeyIvError", "MickeyScalar", "MickeyScalarPacked", "MickeySliced",
    "Mk2Error", "scalar_keystream",
    "mickey_constants", "mickey_sliced_words", "bulk_colmajor", "bulk_rowmajor",
    "words_to_lane_bits", "words_to_lane_bytes", "words_lane_major_bytes",
    "GrainGenerator", "GrainKeyIv", "GrainKeyIvError", "GrainSliced", "grain_sliced_words",
    "grain", "hostmem", "kernels", "mickey", "seedgen", "sharding",
]
