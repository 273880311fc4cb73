#!/usr/bin/env bash
# Static SASS statistics of one trace-kernel instantiation of a built library (no GPU needed):
# registers / spills and the opcode histogram.  Usage: sass_stats.sh <lib.so> <mangled-suffix>
# e.g. the C3 default kernel: Li0ELb0ELi2ELb0ELb0E (CAP none, no steering, fast pow2 sampler)
set -eu
lib=$(realpath "$1"); pat=${2:-Li0ELb0ELi2ELb0ELb0E}; cfg=${CFG:-ILi1ELi1ELi4ELi8ELi128ELb1ELi4ELb1ELi1EEE}
d=$(mktemp -d); trap 'rm -rf $d' EXIT
(cd $d && cuobjdump -xelf phg_trace.sm_100a.cubin "$lib" >/dev/null)
nvdisasm -c $d/phg_trace.sm_100a.cubin > $d/all.sass
name=$(grep -o "^\.text\._ZN3phg12trace_kernelINS_3Cfg${cfg}${pat}[^:]*" $d/all.sass | head -1)
awk -v n="$name:" '$0==n{on=1;next} on && /^\.text\./{exit} on' $d/all.sass > $d/k.sass
cuobjdump -res-usage "$lib" 2>/dev/null | grep -A1 "${name#.text.}" | tail -1
echo "static instructions: $(grep -cE '^\s+/\*[0-9a-f]+\*/' $d/k.sass)"
grep -oE "^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T] )?[A-Z0-9_.]+" $d/k.sass | awk '{print $NF}' | sed 's/\..*//' \
  | sort | uniq -c | sort -rn | head -${TOP:-25} | tr '\n' ' '; echo
[ -n "${KEEP:-}" ] && cp $d/k.sass "$KEEP"
true
