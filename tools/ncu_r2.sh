#!/bin/bash
# Round-2 ncu --set full captures of steady-state launches (one bench step
# each, python bench.py --ncu); reports land in gpurun_out/prof_r2_<name>.ncu-rep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cap() {  # name regex skip count
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$2" -s "$3" -c "$4" -o "gpurun_out/prof_r2_$1" -f python bench.py --ncu \
    > "gpurun_out/ncu_r2_$1.log" 2>&1
  echo "ncu $1 exit $?"
  # keep the results small enough to travel back (gpurun_out <= 64 MiB)
  ncu -i "gpurun_out/prof_r2_$1.ncu-rep" --page raw --csv > "gpurun_out/prof_r2_$1_raw.csv" 2>/dev/null
  ncu -i "gpurun_out/prof_r2_$1.ncu-rep" --page details --csv > "gpurun_out/prof_r2_$1_details.csv" 2>/dev/null
  [ -n "$KEEP_REP" ] || rm -f "gpurun_out/prof_r2_$1.ncu-rep"
}
for spec in "$@"; do
  IFS=: read -r name re skip count <<< "$spec"
  cap "$name" "$re" "$skip" "$count"
done
