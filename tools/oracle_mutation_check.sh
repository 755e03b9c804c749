#!/bin/bash
# Mutation check of the oracle pins (round-1 review, "Next round" item 1):
# each mutation below is a plausible slip in the oracle (a swapped axis, a
# wrong child or time offset, a misplaced flux memory, a sign, a constant).
# For each one a mutated copy of the oracle is built under /tmp and the pins
# (tests/test_oracle_pins_r2.py + the older AMR / physics pins) are run against
# it through ORACLE_LIB.  Every mutation must make at least one pin fail.
# Usage: tools/oracle_mutation_check.sh [log]   (CPU only, ~2 min)
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
LOG=${1:-$ROOT/profiles/round2_oracle_mutations.log}
W=$(mktemp -d /tmp/orcmut.XXXXXX)
TESTS="tests/test_oracle_pins_r2.py tests/test_oracle_amr.py tests/test_oracle_physics.py tests/test_oracle_tables.py"
: > "$LOG"
# name | file | python-literal old | python-literal new
MUTS=(
"projection: child offset on the wrong axis|ader_oracle_amr.c|xi[k] = (off[k] + gq[gi[k]]) / r;|xi[k] = (off[(k + 1) % d] + gq[gi[k]]) / r;"
"projection: time fraction reversed|ader_oracle_amr.c|else orc_eval_st(d, M, nv, poly, xi, tau, val);|else orc_eval_st(d, M, nv, poly, xi, 1.0 - tau, val);"
"coarse-fine: tangential offset from the wrong axis|ader_oracle_amr.c|offK[k] = (double)(C->idx[k] % r) / r;|offK[k] = (double)(C->idx[(k + 1) % d] % r) / r;"
"coarse-fine: sub-interval offset m+1|ader_oracle_amr.c|double toff = (double)m / r, tscl = 1.0 / r;|double toff = (double)(m + 1) / r, tscl = 1.0 / r;"
"coarse-fine: sub-interval scale 1|ader_oracle_amr.c|double toff = (double)m / r, tscl = 1.0 / r;|double toff = (double)m / r, tscl = 1.0;"
"flux memory: deposited on the wrong face|ader_oracle_amr.c|int face = 2 * dir + (side ? 0 : 1);|int face = 2 * dir + side;"
"flux memory: children of the face taken with x/y swapped|ader_oracle_amr.c|    int off[3] = {q % r, (q / r) % r, (d == 3) ? q / (r * r) : 0};\n    if (off[dir]|    int off[3] = {(q / r) % r, q % r, (d == 3) ? q / (r * r) : 0};\n    if (off[dir]"
"flux memory: normalised by r^(d-1)|ader_oracle_amr.c|F[v] = F[v] / (double)A->rd;|F[v] = F[v] / (double)(A->rd / A->r);"
"MHD: induction row sign|ader_oracle.c|f[5 + k] = v[dir] * B[k] - B[dir] * v[k]|f[5 + k] = v[dir] * B[k] + B[dir] * v[k]"
"MHD: Psi missing from the normal induction row|ader_oracle.c|(k == dir ? u[8] : 0.0);|(k == dir ? 0.0 : 0.0);"
"MHD: energy flux v.B term with 8 pi|ader_oracle.c|f[4] = v[dir] * (u[4] + pt) - B[dir] * vB / (4.0 * M_PI);|f[4] = v[dir] * (u[4] + pt) - B[dir] * vB / (8.0 * M_PI);"
"MHD: GLM row c_h instead of c_h^2|ader_oracle.c|f[8] = ch * ch * B[dir];|f[8] = ch * B[dir];"
"WENO: exponent r = 6|ader_oracle.c|pow(sig + 1e-14, 8.0)|pow(sig + 1e-14, 6.0)"
"WENO: eps = 1e-12|ader_oracle.c|pow(sig + 1e-14, 8.0)|pow(sig + 1e-12, 8.0)"
"WENO: eps = 1e-16|ader_oracle.c|pow(sig + 1e-14, 8.0)|pow(sig + 1e-16, 8.0)"
"WENO: central linear weight 1e3 (M=2)|ader_oracle.c|B->L[0] = M / 2; B->R[0] = M / 2; B->lin[0] = 1e5;|B->L[0] = M / 2; B->R[0] = M / 2; B->lin[0] = 1e3;"
)
fail=0
for m in "${MUTS[@]}"; do
  IFS='|' read -r name file old new <<< "$m"
  rm -rf "$W/src"; cp -r "$ROOT/oracle" "$W/src"; rm -f "$W/src/liboracle.so"
  python - "$W/src/$file" "$old" "$new" <<'EOF'
import sys
p, old, new = sys.argv[1], sys.argv[2].replace("\\n", "\n"), sys.argv[3].replace("\\n", "\n")
s = open(p).read()
assert s.count(old) == 1, f"mutation anchor not found exactly once: {old!r}"
open(p, "w").write(s.replace(old, new))
EOF
  if [ $? -ne 0 ]; then echo "ANCHOR MISSING: $name" | tee -a "$LOG"; fail=1; continue; fi
  make -s -C "$W/src" liboracle.so > /dev/null 2>&1 || { echo "BUILD FAILED: $name" | tee -a "$LOG"; fail=1; continue; }
  out=$(cd "$ROOT" && ORACLE_LIB="$W/src/liboracle.so" timeout 900 python -m pytest $TESTS -q -m "not gpu" -p no:randomly 2>&1 | tail -40)
  nfail=$(echo "$out" | grep -c "^FAILED")
  if [ "$nfail" -gt 0 ]; then
    echo "CAUGHT ($nfail pins fail): $name" | tee -a "$LOG"
    echo "$out" | grep "^FAILED" | sed 's/ - .*//' | head -6 | sed 's/^/    /' >> "$LOG"
  else
    echo "NOT CAUGHT: $name" | tee -a "$LOG"; fail=1
  fi
done
rm -rf "$W"
echo "mutation check: $([ $fail -eq 0 ] && echo all caught || echo SOME NOT CAUGHT)" | tee -a "$LOG"
exit $fail
