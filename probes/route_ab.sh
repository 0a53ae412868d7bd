#!/bin/bash
# routing at decode sizes (samoyeds_route per call in a CUDA graph).  Round-2
# variants tried against this path and removed: one 1024-thread
# block for top-k + compaction, top-k by warp-argmax rounds, one cooperative
# launch with a grid barrier -- all slower at T = 64, E = 64.
python probes/route_probe.py
