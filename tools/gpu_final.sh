#!/bin/bash
# Round-end style validation: the driver's commands, in its order.
cd "$(dirname "$0")/.."
O=gpurun_out/final
mkdir -p $O
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
( time timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > $O/ref.json 2> $O/ref.err
( time timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 ) > $O/bench.json 2> $O/bench.err
