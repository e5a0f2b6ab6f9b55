"""SFCT tensor files (the reference's container, proj/src/tensor.cpp:17-64) for the Python
side: magic b"SFCT0001", little-endian u32 header length, compact JSON header with sorted keys
{"dtype":"f64","layout":"row-major-nchw","shape":[...]}, then the raw little-endian doubles.
Byte-identical to what the C++ drop-in's sfconv::save_sfct writes.  Host I/O only."""
import json
import struct

import numpy as np

MAGIC = b"SFCT0001"


def save_sfct(path, tensor) -> None:
    """Write any array-like (numpy / torch, any device) as an fp64 SFCT file."""
    if hasattr(tensor, "detach"):
        tensor = tensor.detach().cpu().numpy()
    a = np.ascontiguousarray(tensor, dtype="<f8")
    header = json.dumps({"dtype": "f64", "layout": "row-major-nchw", "shape": [int(d) for d in a.shape]},
                        separators=(",", ":"), sort_keys=True).encode()
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<I", len(header)))
        f.write(header)
        f.write(a.tobytes())


def load_sfct(path) -> np.ndarray:
    """Read an SFCT file; raises RuntimeError with the reference's messages on bad input."""
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError(f"cannot open: {path}") from None
    with f:
        if f.read(8) != MAGIC:
            raise RuntimeError(f"not an SFCT file: {path}")
        lb = f.read(4)
        if len(lb) != 4:
            raise RuntimeError(f"truncated SFCT header: {path}")
        (hlen,) = struct.unpack("<I", lb)
        hs = f.read(hlen)
        if len(hs) != hlen:
            raise RuntimeError(f"truncated SFCT header: {path}")
        header = json.loads(hs)
        if header["dtype"] != "f64":
            raise RuntimeError(f"unsupported SFCT dtype: {header['dtype']}")
        if header["layout"] != "row-major-nchw":
            raise RuntimeError("unsupported SFCT layout")
        shape = tuple(int(d) for d in header["shape"])
        n = int(np.prod(shape, dtype=np.int64)) if shape else 1
        payload = f.read(8 * n)
        if len(payload) != 8 * n:
            raise RuntimeError(f"truncated SFCT payload: {path}")
    return np.frombuffer(payload, dtype="<f8").reshape(shape).astype(np.float64)
