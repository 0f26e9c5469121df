#!/bin/bash
# One entry point for the gpurun jobs this repo runs (replaces the per-experiment
# scratch scripts): tools/gpu_tasks.sh <task> [args]. Outputs go to gpurun_out/.
#   check            pytest -m gpu + smoke() (the round-end gate)
#   bench [N]        bench.py at N GPUs (torchrun for N > 1) + the reference arm
#   launches         ncu launch list (gpu__time_duration) of a short bench run
#   ncu <regex> [n]  one --set full capture of the n-th launch of kernels matching regex
#   epi <args>       tools/epi_probe.py (SPHEMU_TC_DBG / SPHEMU_TC_CG from the env)
#   sweep <N> <VARIANT> <HP> <k=v,..>  tools/ab.py at order N under each environment assignment
#                    (e.g. sweep 32400 dpsp fp16 SPHEMU_RESERVE_EARLY=8,SPHEMU_RESERVE_EARLY=16)
#   timeline <N> <VARIANT>   chain/bulk stream busy and idle times (tools/chol_timeline.py, timeline_gaps.py)
#   oz               the INT8 DP-update kernel alone (tools/micro/oz_bench, SPHEMU_OZ_DBG 0/1/2) + tools/oz_check.py
#   dist <G> <P> [k=v,..]   tools/dist_perf.py on C3 over G GPUs as P x G/P under each assignment
#                    (k=v+k2=v2 sets several variables for one run)
#   disttl <G> <P>   per-rank phase totals of the distributed factorization (tools/dist_timeline.py)
# The round-2 experiments behind the numbers in DESIGN.md were these tasks with the
# settings quoted there.
set -u
mkdir -p gpurun_out
task=${1:-check}; shift || true
case "$task" in
  check)
    timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "PYTEST_EXIT $?" >> gpurun_out/pytest_gpu.log
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "SMOKE_EXIT $?" >> gpurun_out/smoke.log
    tail -n 3 gpurun_out/pytest_gpu.log; tail -n 3 gpurun_out/smoke.log ;;
  bench)
    n=${1:-1}
    if [ "$n" = 1 ]; then
      timeout 1200 python bench.py --steps ${STEPS:-20} --warmup ${WARMUP:-5} > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
      timeout 1200 python bench.py --impl reference --steps ${STEPS:-20} --warmup ${WARMUP:-5} > gpurun_out/bench_ref_n1.json 2> gpurun_out/bench_ref_n1.err
    else
      timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps ${STEPS:-3} --warmup ${WARMUP:-3} > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
    fi
    echo "EXIT $?"; tail -c 3000 gpurun_out/bench_n$n.json ;;
  launches)
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${COUNT:-20000} --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launches.log 2>&1; echo "EXIT $?" ;;
  ncu)
    timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$1" -s ${2:-5} -c 1 -o gpurun_out/ncu_${NAME:-kernel} -f python ${SCRIPT:-bench.py} ${SCRIPT_ARGS:---steps 1 --warmup 3} > gpurun_out/ncu_${NAME:-kernel}.log 2>&1; echo "EXIT $?" ;;
  epi)  # the SPHEMU_TC_DBG modes exist only in a diagnostics build
    make -C paper_2408_04440_b200/csrc DIAG=1 -B -j8 > /dev/null
    python tools/epi_probe.py "$@" ;;
  sweep)
    n=$1; v=$2; hp=$3; IFS=',' read -ra sets <<< "${4:-NONE=1}"
    for kv in "${sets[@]}"; do echo "$kv"; env ${kv//+/ } timeout 300 python tools/ab.py "$n" "$v" "$hp" ${REPS:-3} ${TILE:-512}; done ;;
  timeline)
    timeout 600 python tools/chol_timeline.py "$1" ${TILE:-512} "$2" ${HP:-fp16} 2>/dev/null | head -9
    timeout 600 python tools/timeline_gaps.py "$1" "$2" ${HP:-fp16} ;;
  oz)  # the SPHEMU_OZ_DBG modes exist only in a diagnostics build
    make -C paper_2408_04440_b200/csrc DIAG=1 -B -j8 > /dev/null
    tools/micro/build_oz_bench.sh
    for d in 0 1 2; do echo "SPHEMU_OZ_DBG=$d"; SPHEMU_OZ_DBG=$d timeout 60 ./tools/micro/oz_bench; done
    timeout 900 python tools/oz_check.py 4096 512 ;;
  dist|disttl)
    g=$1; p=$2; IFS=',' read -ra sets <<< "${3:-NONE=1}"
    script=tools/dist_perf.py; [ "$task" = disttl ] && script=tools/dist_timeline.py
    for kv in "${sets[@]}"; do echo "$kv"
      env ${kv//+/ } timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$g" --master-addr 127.0.0.1 \
        --master-port 29533 $script ${N:-129600} 512 ${VARIANT:-dpsphp} ${HP:-bf16} "$p" ${W0:-100} 2>&1 | grep -v "^W\|Warn\|return func\|\*\*\*"
    done ;;
  *)
    echo "unknown task $task"; exit 2 ;;
esac
