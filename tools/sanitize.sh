#!/bin/bash
# compute-sanitizer over a reduced -m gpu subset that covers K1 (SELL
# iterate, heavy combine, narrow, ones step), K2 (cooperative select with the
# fused split, small check, finish, publish; RANKING certificates and the
# cached-pair speculation with page-locked verdicts), the device-driven TOPK
# loop (kernels queued behind a converged check), K3, K4 (dynamic repair,
# heavy-row routes) and the fused NVLink-store exchange through real CUDA
# IPC mappings (two processes).  Logs: gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
SEL="tests/test_gpu_parity.py::test_small_golden_cases_bitwise \
tests/test_gpu_parity.py::test_rmat_s12_topk_vs_oracle \
tests/test_gpu_parity.py::test_grid256_ranking_bitwise \
tests/test_gpu_parity.py::test_iterate_and_check_step_by_step \
tests/test_gpu_parity.py::test_directed_graph_and_pair_score \
tests/test_gpu_dynamic.py::test_golden_dynamic_sequences \
tests/test_gpu_dynamic.py::test_heavy_row_repair_routes_bitwise \
tests/test_gpu_distributed.py::test_cuda_shards_equal_single_gpu \
tests/test_gpu_distributed.py::test_fused_exchange_two_processes_ipc"
for tool in memcheck racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --target-processes all --error-exitcode 99 \
      --print-limit 200 python -m pytest -q -x $SEL > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
done
