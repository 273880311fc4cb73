# build an experiment library: bexp.sh <dir> [nvcc flags...]
cd /root/repo
d=$1; shift
python - "$d" "$@" <<'PY'
import sys, json
from paper_2604_05794_b200 import build
build.build(force=True, extra=sys.argv[2:], out=sys.argv[1] + "/libphg_b200.so")
PY
profiles/sass_stats.sh $d/libphg_b200.so
