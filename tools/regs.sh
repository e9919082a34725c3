# register / spill summary of one build: bash tools/regs.sh <src-root> <out.txt> [kernel-regex]
R=${1:-.}; O=${2:-/tmp/regs.txt}
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false \
  -Xcompiler -fPIC -shared -Xptxas=-v -o /tmp/regs_lib.so $R/paper_2601_12241_b200/csrc/padsim.cu \
  $R/paper_2601_12241_b200/csrc/controller_host.cpp > $O.raw 2>&1
python3 - $O.raw ${3:-.} > $O <<'PY'
import re, sys
cur = None
for l in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", l)
    if m: cur = m.group(1); continue
    m = re.search(r"Used (\d+) registers", l)
    if m and cur and re.search(sys.argv[2], cur):
        sp = re.search(r"(\d+) bytes spill", l)
        print(cur, m.group(1))
PY
