#!/bin/bash
# Does a process exit after smoke()? Each variant runs with a deadline; a process still alive
# at the deadline gets its threads' kernel stacks / wchan / syscalls dumped, then is killed.
mkdir -p gpurun_out
run() {
  label=$1; shift
  ( env "$@" python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/xd_$label.log 2>&1 ) &
  local sub=$!
  sleep 2
  local pid=$(pgrep -P $sub python | head -1)
  for i in $(seq 1 90); do
    kill -0 $sub 2>/dev/null || { echo "$label: exited (${i}s)" >> gpurun_out/xd_summary.txt; return; }
    sleep 1
  done
  echo "$label: HUNG (pid $pid)" >> gpurun_out/xd_summary.txt
  for t in /proc/$pid/task/*; do
    echo "--- $t $(cat $t/comm) wchan=$(cat $t/wchan)" >> gpurun_out/xd_$label.stacks
    cat $t/syscall >> gpurun_out/xd_$label.stacks 2>&1
    cat $t/stack >> gpurun_out/xd_$label.stacks 2>&1
  done
  kill -9 $pid 2>/dev/null
  wait $sub 2>/dev/null
}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/xd_build.log 2>&1
run plain GACE_X=0
run nojit GACE_JIT=0
run sync_layout GACE_JIT_LAYOUT=0
run minrows GACE_JIT_MIN_ROWS=1000000000
cat gpurun_out/xd_summary.txt
