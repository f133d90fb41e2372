"""B200-native (sm_100a) data-parallel core of the Modified No Search fractal coder
(arXiv 1501.02894), a drop-in for the reference ``mnscodec`` encode/decode hot path.

Public API mirrors mnscodec (same names, signatures, dataclasses, error messages):
encode_quadtree, try_phase1, try_phase2, decode, decode_step, encode_full_search, encode_local_search,
write_stream, read_stream, stream_bit_count, plus the device layer used by
bench.py and the multi-GPU sharding (encode_device, decode_device, ...).
"""

from .types import (  # noqa: F401
    CONTRAST_SETS,
    CONTRAST_VALUES,
    DELTA_MAGNITUDE_BITS,
    LEVEL_SIZES,
    MODES,
    ROOT_SIZE,
    BaselinePayload,
    BlockRect,
    DecodeConfig,
    EncoderConfig,
    GrayImage,
    LeafRecord,
    Phase1Payload,
    Phase2Payload,
    QuadtreeCode,
    delta_limit,
    dequantize_contrast,
    round_to_int,
)
from .codec import (  # noqa: F401
    DeviceCode,
    build_unit_map,
    co_domain_rect,
    decode,
    decode_device,
    decode_step,
    encode_device,
    encode_full_search,
    encode_local_search,
    encode_quadtree,
    full_search_device,
    local_search_device,
    pad_to_multiple,
    try_phase1,
    try_phase2,
    write_stream_device,
)

from . import bitstream  # noqa: F401  (reference mnscodec.bitstream)
from .bitstream import (  # noqa: F401
    StreamFormatError,
    leaf_bit_width,
    level_id_bit_count,
    payload_bit_width,
    read_stream,
    stream_bit_count,
    write_stream,
)
from .rd import (  # noqa: F401  (reference mnscodec.bench)
    RD_CSV_COLUMNS,
    OffsetHistogram,
    RdPoint,
    histogram_csv,
    mse,
    psnr,
    offset_histogram,
    offset_histogram_device,
    rd_csv,
    rd_sweep,
)

__version__ = "0.1.0"
