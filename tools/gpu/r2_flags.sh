# C3 timing of compile-flag variants of the engine (built on the box)
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
cd paper_2504_03887_b200/csrc
B="nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -I../../include -shared replay.cu"
$B -Xptxas --allow-expensive-optimizations=true -o /tmp/v1.so &
$B -Xptxas --register-usage-level=10 -o /tmp/v2.so &
$B -Xptxas --register-usage-level=0 -o /tmp/v3.so &
wait
cd ../..
for v in default /tmp/v1.so /tmp/v2.so /tmp/v3.so default; do
  echo "== $v"
  if [ "$v" = default ]; then a=""; else a="--lib $v"; fi
  timeout 300 python tools/prof_replay.py --traces 10000 --launches 4 $a 2>&1 | tail -2
done
