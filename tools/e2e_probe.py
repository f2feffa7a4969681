"""The bench's e2e leg alone (tec_eval_fused_conv on host buffers, C1-C12
b64): python tools/e2e_probe.py [f32tc|bf16|i8] [steps]."""
import json
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

compute = sys.argv[1] if len(sys.argv) > 1 else "f32tc"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
r = bench.run_e2e(types.SimpleNamespace(steps=steps), 64, 0, compute, 1)
r["chunk_kb"] = os.environ.get("TEC_SM100_CHUNK_KB", "default")
print(json.dumps(r))
