#!/bin/bash
# Host-logic check of the N > 1 bench path on a one-GPU box: torchrun with 2
# ranks, both on cuda:0, gloo collectives (--functional-1gpu).  Not a
# measurement.  The line's checksum must equal the 1-GPU line's (strong
# scaling over one configs[2] image).
set -u
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
python bench.py --steps 3 --warmup 3 --no-extras --no-e2e --no-cpu-baseline > gpurun_out/fn_n1.json 2> gpurun_out/fn_n1.err; echo "n1 rc=$?"
$R bench.py --gpus 2 --steps 3 --warmup 3 --no-extras --functional-1gpu > gpurun_out/fn_n2.json 2> gpurun_out/fn_n2.err; echo "n2 rc=$?"
$R bench.py --gpus 2 --kernel window --steps 3 --warmup 3 --functional-1gpu > gpurun_out/fn_n2_window.json 2> gpurun_out/fn_n2_window.err; echo "n2 window rc=$?"
# (--halo exchange is not run here: gloo cannot send CUDA tensors point to point; its logic is
# covered by tests/test_dist_gloo.py on CPU tensors, and NCCL sends device memory)
python bench.py --kernel window --steps 3 --warmup 3 > gpurun_out/fn_n1_window.json 2> gpurun_out/fn_n1_window.err; echo "n1 window rc=$?"
$R bench.py --gpus 2 --impl reference --steps 1 --warmup 1 > gpurun_out/fn_n2_ref.json 2> gpurun_out/fn_n2_ref.err; echo "n2 ref rc=$?"
python - <<'PY'
import json
a = json.load(open("gpurun_out/fn_n1.json")); b = json.load(open("gpurun_out/fn_n2.json"))
print("checksum n1", a["checksum"], "n2", b["checksum"], "equal", a["checksum"] == b["checksum"],
      "counts", a["status_counts"] == b["status_counts"], "n_gpus", b["n_gpus"], "workload", b["config"]["workload"])
print("n2 e2e", b.get("e2e", {}).get("value"), "cpu_baseline", "cpu_baseline" in b)
c = json.load(open("gpurun_out/fn_n1_window.json")); d = json.load(open("gpurun_out/fn_n2_window.json"))
print("window checksum n1", c["checksum"], "n2", d["checksum"], "equal", c["checksum"] == d["checksum"])

PY
