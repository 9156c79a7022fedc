#!/bin/bash
# compute-sanitizer over the library's kernels on a small cloud (tools/sanitize_case.py:
# neighbor build, tile planning, tcgen05 bf16 / split kernels, exact engines).
# Usage on a GPU box: tools/sanitize.sh [outdir].  Exit 0 iff
#   memcheck, synccheck, initcheck: 0 errors;
#   racecheck over every kernel except the tcgen05 pipelines: 0 hazards.
# The tcgen05 pipelines hand shared-memory slots between warps through
# mbarriers that the tensor core arrives on (tcgen05.commit), which racecheck
# cannot see; their racecheck run is reported separately (hazard sites summed
# per kernel and instruction) and not gated.
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=${1:-$ROOT/gpurun_out}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
TC='regex=k_conv_(fwd_tc|bwd_fused|wgrad_tc)'
export SAN_POINTS=${SAN_POINTS:-3000}
rc=0
run() {  # name, extra args...
  local name=$1; shift
  timeout 1500 $CS "$@" --print-limit ${SAN_PRINT:-1000} --target-processes all python "$ROOT/tools/sanitize_case.py" \
    > "$OUT/sanitize_$name.log" 2>&1
  local ok=$(grep -c 'SANITIZE CASE OK' "$OUT/sanitize_$name.log")
  echo "$name: $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' "$OUT/sanitize_$name.log" | tail -1) case_ok=$ok"
  [ "$ok" = 1 ] || rc=1
}
for tool in ${SAN_TOOLS:-memcheck synccheck initcheck}; do
  run $tool --tool $tool
  grep -q "ERROR SUMMARY: 0 errors" "$OUT/sanitize_$tool.log" || rc=1
done
run racecheck_non_tc --tool racecheck --racecheck-report hazard --kernel-name-exclude "$TC"
grep -q "RACECHECK SUMMARY: 0 hazards" "$OUT/sanitize_racecheck_non_tc.log" || rc=1
[ "${SAN_TC:-1}" = 1 ] && for k in fwd_tc bwd_fused wgrad_tc; do
SAN_MATH=bf16 SAN_PRINT=3000 run racecheck_$k --tool racecheck --racecheck-report hazard --kernel-name "regex=k_conv_$k"
python3 - "$OUT/sanitize_racecheck_$k.log" "k_conv_$k" <<'PY'
import re, sys, collections
c = collections.Counter(); kern = None; kind = None; sites = []
for line in open(sys.argv[1], errors="replace"):
    m = re.search(r"Potential (\w+) hazard", line)
    if m: kind, sites = m.group(1), []
    m = re.search(r"(Read|Write) Thread .* at (npcg::\S+?)\(", line)
    if m: sites.append(m.group(1) + " " + m.group(2).split("::")[-1])
    if kind and "Saved host backtrace" in line:
        c[(sys.argv[2], kind, " / ".join(sorted(sites)))] += 1; kind = None
for (k, t, s), n in c.most_common(20): print(f"  tc hazard sites (of the first 3000): {n:5d}  {k}  {t}  {s}")
PY
done
exit $rc
