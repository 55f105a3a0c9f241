"""c5 PiTSBiCG time-to-tolerance (full size; ~minutes)."""
import json
import sys
sys.path.insert(0, ".")
import bench  # noqa: E402

r = bench.device_time_to_tolerance("c5")
print(json.dumps(r))
