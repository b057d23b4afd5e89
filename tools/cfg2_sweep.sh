#!/bin/bash
# cfg2 engine step under leaf-GEMM caps, skews and priority modes (device-resident)
for cap in 0 8 16 32; do for skew in 0 1; do for pm in 2 3; do
  r=$(BI_LEAF_GEMM_CAP=$cap BI_ENGINE_SKEW=$skew BI_PRIORITY_MODE=$pm timeout 120 python tools/ab_time.py --cfg2-only 2>&1 | tail -1)
  echo "cap=$cap skew=$skew pm=$pm $r"
done; done; done
