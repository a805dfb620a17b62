mkdir -p gpurun_out
( python scripts/probe_tail.py 2
  FM_CHUNK_FINE_DRAWS=32 python scripts/probe_tail.py 2
  FM_CHUNK_LANE_DRAWS=256 python scripts/probe_tail.py 2
  FM_TAIL_FACTOR=4 FM_CHUNK_FINE_DRAWS=32 python scripts/probe_tail.py 2
  python scripts/probe_tail.py 3 ) 2>&1 | tee gpurun_out/ab6.txt
