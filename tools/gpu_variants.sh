# build libqem variants (-D...) and time a config with each: CFG=4 bash tools/gpu_variants.sh "QEM_X=0" "QEM_X=4" ...
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in "$@"; do
  python -c "from paper_2503_08264_b200 import build; build.build(defines=('$v',), out='/tmp/qem_$v.so')" > /dev/null 2>&1 || echo "build $v failed"
done
for v in "$@"; do
  echo "== $v"
  QEM_LIB_OVERRIDE=/tmp/qem_$v.so timeout 300 python bench.py --config ${CFG:-5} --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k: round(v,4) for k,v in d['roofline']['kernels_ms'].items()}, round(d['roofline']['frac'],4))"
done
