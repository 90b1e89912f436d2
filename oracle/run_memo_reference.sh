#!/usr/bin/env bash
# One offline run of the UNMODIFIED reference at a BASELINE config too large
# for a single core in one session (c2: 8-12 h serial).
# TEST INFRASTRUCTURE ONLY.
#
# The independent per-subdomain / per-W-column work is spread over worker
# processes that fill a content-hash cache of the reference's own
# dense_sym_eig / generalized_sym_eig / pcg results (oracle/memo.cpp); a final
# ordinary ref_driver run then replays the stock composition
# (ProblemContext + run_with_context, harness.cpp:63-139) end to end with
# every cached call bit-identical to recomputation, times the stock H3 apply
# loop, and exports goldens.  Serial reference setup time = sum of the
# per-entry seconds stored in the cache (reported by summarize in
# tests/golden/make_c2_reference_golden.py).
#
#   oracle/run_memo_reference.sh <config> <workdir> [driver flags...]
set -euo pipefail
cfg=$1; work=$2; shift 2
flags=("$@")
here=$(cd "$(dirname "$0")" && pwd)
drv=$here/_ref/ref_driver_memo
mkdir -p "$work/memo"
cd "$work"
if [ ! -f "$cfg.mtx" ]; then
  python -c "import sys; sys.path.insert(0, '$here/..'); from paper_2106_10913_b200 import problems as P; P.make('$cfg').write('$cfg')"
fi
export AWG_MEMO_DIR=$PWD/memo AWG_MEMO_PCG=1
run_phase() {  # phase nworkers
  local pids=()
  for ((w = 0; w < $2; w++)); do
    "$drv" "$cfg" junk "${flags[@]}" --phase "$1" --worker $w --nworkers "$2" > "phase_$1_$w.log" 2>&1 &
    pids+=($!)
  done
  for p in "${pids[@]}"; do wait "$p"; done
  echo "$(date +%T) phase $1 done"
}
NB=${NB:-8}; NP=${NP:-6}; NW=${NW:-5}
run_phase bs "$NB"
run_phase pencil "$NP"
run_phase w "$NW"
"$drv" "$cfg" out "${flags[@]}" --apply-reps ${APPLY_REPS:-20} > replay.log 2>&1
echo "$(date +%T) replay done"
