#!/usr/bin/env bash
# One-GPU measurement session: full GPU test suite, smoke, the default bench line, the ncu
# launch list of a short bench, one ncu --set full capture of the sync-only comm kernel.
T=${TAG:-r2m}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 3 --warmup 3 --skip-cpu --skip-layerwise --skip-e2e > gpurun_out/${T}_ncu_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_comm|k_update_stream' -s 2 -c 1 -f -o gpurun_out/${T}_kcomm \
  python tools/debug_sync.py resnet50 148 > gpurun_out/${T}_ncu_full.log 2>&1
