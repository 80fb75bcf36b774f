#!/usr/bin/env python
"""NVLink byte counters of one GPU through NVML (nvidia-ml-py), for link-traffic evidence of
the multi-GPU path (achieved NVLink bytes vs the algorithmic bytes; ncu cannot
capture a multi-rank kernel).

`read(dev)` returns {"tx": bytes, "rx": bytes} summed over the GPU's NVLinks (data payload
counters NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX, KiB; falls back to the per-link
COUNT_XMIT/RCV_BYTES fields), or None when NVML or the counters are unavailable.

  python tools/nvlink_counters.py            # print every GPU's counters (probe)
"""
import sys

_FI_DATA_TX, _FI_DATA_RX = 138, 139       # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_{TX,RX} (KiB)
_FI_XMIT_BYTES, _FI_RCV_BYTES = 202, 204  # NVML_FI_DEV_NVLINK_COUNT_{XMIT,RCV}_BYTES (per link)
_MAX_LINKS = 18
_h = {}


def _handle(dev):
    import pynvml
    if not _h:
        pynvml.nvmlInit()
    if dev not in _h:
        _h[dev] = pynvml.nvmlDeviceGetHandleByIndex(dev)
    return _h[dev]


def _fields(h, ids):
    import pynvml
    vals = pynvml.nvmlDeviceGetFieldValues(h, ids)
    out = []
    for v in vals:
        if v.nvmlReturn != 0:
            out.append(None)
        else:
            out.append(int(v.value.ullVal))
    return out


def read(dev):
    """Cumulative NVLink data bytes {tx, rx} of GPU `dev` (physical index), or None."""
    try:
        h = _handle(dev)
        # throughput counters, all links (scopeId UINT_MAX) then per link
        tx, rx = _fields(h, [(_FI_DATA_TX, 0xFFFFFFFF), (_FI_DATA_RX, 0xFFFFFFFF)])
        if tx is not None and rx is not None and (tx or rx):
            return {"tx": tx * 1024, "rx": rx * 1024, "field": "THROUGHPUT_DATA (all links)"}
        ids = [(_FI_DATA_TX, l) for l in range(_MAX_LINKS)] + [(_FI_DATA_RX, l) for l in range(_MAX_LINKS)]
        v = _fields(h, ids)
        if any(x for x in v if x):
            return {"tx": sum(x or 0 for x in v[:_MAX_LINKS]) * 1024, "rx": sum(x or 0 for x in v[_MAX_LINKS:]) * 1024,
                    "field": "THROUGHPUT_DATA (per link)"}
        ids = [(_FI_XMIT_BYTES, l) for l in range(_MAX_LINKS)] + [(_FI_RCV_BYTES, l) for l in range(_MAX_LINKS)]
        v = _fields(h, ids)
        if any(x for x in v if x):
            return {"tx": sum(x or 0 for x in v[:_MAX_LINKS]), "rx": sum(x or 0 for x in v[_MAX_LINKS:]),
                    "field": "COUNT_XMIT/RCV_BYTES (per link)"}
    except Exception:
        return None
    return None


if __name__ == "__main__":
    import pynvml
    pynvml.nvmlInit()
    n = pynvml.nvmlDeviceGetCount()
    for d in range(n):
        h = _handle(d)
        print(d, "all-links:", _fields(h, [(_FI_DATA_TX, 0xFFFFFFFF), (_FI_DATA_RX, 0xFFFFFFFF),
                                          (_FI_XMIT_BYTES, 0xFFFFFFFF), (_FI_RCV_BYTES, 0xFFFFFFFF)]))
        print(d, "per-link DATA_TX:", _fields(h, [(_FI_DATA_TX, l) for l in range(_MAX_LINKS)]))
        print(d, "per-link XMIT_BYTES:", _fields(h, [(_FI_XMIT_BYTES, l) for l in range(_MAX_LINKS)]))
        print(d, "read():", read(d))
    sys.exit(0)
