#!/bin/bash
# Round-2 ncu evidence (run on the GPU box through gpurun; reports land in gpurun_out/, the tracked
# summaries are made from them by scripts/make_profile_summary.py r2 + scripts/ncu_key.py).
# usage: scripts/capture_r2.sh [launches] [scan] [edge] [havoc] [small] [sparse]   (default: all)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
what="${*:-launches scan edge edge_flat edge_flat_large edge_launches havoc small sparse}"
NCU="ncu --clock-control none"
for w in $what; do
  case $w in
    launches)
      $NCU --metrics gpu__time_duration.sum -c 6000 --csv --log-file gpurun_out/r2_bench_launches.csv \
        python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e-dense --e2e-steps 1 --no-harness --no-check \
        > gpurun_out/r2_bench_launches.log 2>&1 ;;
    scan)
      $NCU --set full --import-source on -k regex:hfz_k_scan -s 4 -c 1 -f -o gpurun_out/r2_scan \
        python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-configs --no-harness --no-stress --no-check \
        > gpurun_out/r2_scan.log 2>&1 ;;
    edge)         # the per-exec kernel alone (round 1's design; now only execs whose launches differ in geometry)
      EDGE_N=1024 EDGE_FLAT=0 $NCU --set full --import-source on -k regex:hfz_k_edge_record -s 2 -c 1 -f -o gpurun_out/r2_edge \
        python scripts/probe_k1k3.py edge > gpurun_out/r2_edge.log 2>&1 ;;
    edge_flat)    # the flat path's three kernels
      EDGE_N=1024 $NCU --set full --import-source on -k "regex:hfz_k_edge_(classify|divergent|count)" -s 3 -c 3 -f -o gpurun_out/r2_edge_flat \
        python scripts/probe_k1k3.py edge > gpurun_out/r2_edge_flat.log 2>&1 ;;
    edge_flat_large)
      EDGE_N=1024 EDGE_S=262144 $NCU --set full --import-source on -k "regex:hfz_k_edge_(classify|divergent|count)" -s 3 -c 3 -f -o gpurun_out/r2_edge_flat_large \
        python scripts/probe_k1k3.py edge > gpurun_out/r2_edge_flat_large.log 2>&1 ;;
    edge_launches)
      EDGE_N=1024 $NCU --metrics gpu__time_duration.sum -k regex:hfz_k_edge -c 15 python scripts/probe_k1k3.py edge 2>&1 \
        | grep -E "hfz_k_edge|gpu__time" | paste - - | awk '{print $1, $2, $(NF-1), $NF}' > gpurun_out/r2_edge_flat_launches.txt ;;
    havoc)
      $NCU --set full --import-source on -k regex:hfz_k_havoc -s 4 -c 2 -f -o gpurun_out/r2_havoc \
        python scripts/probe_k1k3.py havoc > gpurun_out/r2_havoc.log 2>&1 ;;
    small)
      $NCU --set full --import-source on -k regex:hfz_k_small_step -s 8 -c 1 -f -o gpurun_out/r2_small_step \
        python scripts/probe_small.py > gpurun_out/r2_small_step.log 2>&1 ;;
    sparse)
      $NCU --set full --import-source on -k regex:hfz_k_sparse -s 2 -c 2 -f -o gpurun_out/r2_sparse \
        python scripts/probe_sparse.py --chunks 65536 > gpurun_out/r2_sparse.log 2>&1 ;;
  esac
  echo "capture $w: rc=$?"
done
ls -la gpurun_out/*.ncu-rep
