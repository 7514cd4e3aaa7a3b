#!/bin/bash
# Build the timeline variant of evo_ln_proj.cu (-DLP_TL=1: globaltimer stamps into `mean`) as a
# standalone .so under tools/lpvar/ for tools/lp_timeline.py (the product build never sets LP_TL).
cd "$(dirname "$0")/.."
mkdir -p tools/lpvar
cat > /tmp/lp_stub.cu <<'X'
namespace evo { void set_error_detail(const char*) {} }
X
/usr/local/cuda/bin/nvcc -O3 -std=c++17 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a \
  -Xcompiler -fPIC -shared -DLP_TL=1 -I include -I paper_2404_11068_b200/csrc \
  paper_2404_11068_b200/csrc/evo_ln_proj.cu /tmp/lp_stub.cu -lcuda -o tools/lpvar/lp_tl.so
