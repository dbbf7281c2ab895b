# compute-sanitizer passes over small instances of every kernel family of the
# hot path (one gpurun call); logs under gpurun_out/san/
mkdir -p gpurun_out/san
O=gpurun_out/san
PC="python tools/profile_case.py"
run() {  # name tool command...
  local name=$1 tool=$2; shift 2
  timeout 900 compute-sanitizer --tool $tool --print-limit 30 --error-exitcode 9 "$@" > $O/${tool}_$name.log 2>&1
  echo "$tool $name rc=$? $(grep -c '=========     at ' $O/${tool}_$name.log) sites; $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' $O/${tool}_$name.log | tail -1)"
}
for tool in memcheck racecheck; do
  run smoke    $tool python -c "import __graft_entry__ as g; g.smoke()"
  run k160     $tool $PC --n 6000 --k 160 --nrhs 160 --transpose --p 4
  run k128     $tool $PC --n 6000 --k 128 --nrhs 32 --transpose --p 4
  run k64      $tool $PC --n 6000 --k 64 --nrhs 1 --transpose --p 6
  run k64piv   $tool $PC --n 6000 --k 64 --nrhs 4 --piv --transpose --p 6
  run k160piv  $tool $PC --n 6000 --k 160 --nrhs 16 --piv --transpose --p 4
  run k16      $tool $PC --n 20000 --k 16 --nrhs 1 --transpose
  run k16piv   $tool $PC --n 20000 --k 16 --nrhs 3 --piv --transpose
done
run smoke synccheck python -c "import __graft_entry__ as g; g.smoke()"
run k160 synccheck $PC --n 6000 --k 160 --nrhs 160 --transpose --p 4
run k64piv synccheck $PC --n 6000 --k 64 --nrhs 4 --piv --transpose --p 6
run k160 initcheck $PC --n 6000 --k 160 --nrhs 160 --transpose --p 4
run k16 initcheck $PC --n 20000 --k 16 --nrhs 1 --transpose
ls -la $O
