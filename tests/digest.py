"""digest64 of one pipeline instance (test side; the device computes the same
value in its per-instance stats record, include/recon_b200.h).

  e(tag, i, v) = mix(mix((tag << 48) ^ i) ^ (v & 0xffffffff))
  ok:     digest = mix( sum_i e(1, i, src[i]) + sum_i e(2, i, dst[i]) + sum_j e(3, j, move_batch[j])
                        + e(5, 0, P) + e(6, 0, D & 0xffffffff) + e(7, 0, D >> 32) + e(8, 0, nb) )   (mod 2^64)
  failed: digest = mix( e(4, 0, status) )
mix = splitmix64's finaliser.  Order-sensitive through the index, associative
through the sum, so a device reduction reproduces it.
"""
import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def mix(z):
    z = np.asarray(z, dtype=np.uint64) + _G
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def elem(tag: int, idx, vals):
    idx = np.asarray(idx, dtype=np.uint64)
    v = np.asarray(vals).astype(np.int64).astype(np.uint64) & np.uint64(0xFFFFFFFF)
    return mix(mix((np.uint64(tag) << np.uint64(48)) ^ idx) ^ v)


def _sum(x) -> np.uint64:
    return np.uint64(np.sum(np.asarray(x, dtype=np.uint64), dtype=np.uint64))


def instance_digest(status: int, src, dst, move_batch, total_displacement: int, batch_count: int) -> int:
    with np.errstate(over="ignore"):
        if status != 0:
            return int(mix(elem(4, 0, status)))
        P = len(src)
        D = int(total_displacement)
        acc = np.uint64(0)
        acc += _sum(elem(1, np.arange(P), src))
        acc += _sum(elem(2, np.arange(P), dst))
        acc += _sum(elem(3, np.arange(len(move_batch)), move_batch))
        acc += elem(5, 0, P) + elem(6, 0, D & 0xFFFFFFFF) + elem(7, 0, D >> 32) + elem(8, 0, batch_count)
        return int(mix(acc))


def pipeline_digests(out: dict, count: int, stride_paths: int, move_stride: int) -> np.ndarray:
    """digest64 per instance of a ReconLib.pipeline_batch result."""
    d = np.zeros(count, np.uint64)
    for i in range(count):
        st = int(out["status"][i])
        P = int(out["path_count"][i])
        D = int(out["total_displacement"][i])
        s = out["path_src"][i * stride_paths:i * stride_paths + P]
        t = out["path_dst"][i * stride_paths:i * stride_paths + P]
        mb = out["move_batch"][i * move_stride:i * move_stride + D]
        d[i] = instance_digest(st, s, t, mb, D, int(out["batch_count"][i]))
    return d
