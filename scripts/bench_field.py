#!/usr/bin/env python
"""Run selected secondary fields of bench.py on their own (dev tool: one JSON line per field).

  python scripts/bench_field.py cfg5_mla_expanded cfg5_mla
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

FIELDS = {"block16": bench.secondary_block16, "cfg3_llama70b": bench.secondary_cfg3,
          "cfg4_longctx": bench.secondary_cfg4, "cfg5_mla": bench.secondary_cfg5,
          "cfg5_mla_expanded": bench.secondary_cfg5_expanded, "fp8_kv": bench.secondary_fp8}


def main():
    args = bench.parse([])
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    pk = bench.peaks()
    for name in sys.argv[1:]:
        rec = FIELDS[name](args, dev, pk)
        print(json.dumps({"field": name, **rec}), flush=True)


if __name__ == "__main__":
    main()
