# the driver's default invocations: bench.py and bench.py --impl reference with no flags
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
S=$SECONDS; python bench.py > gpurun_out/bare.log 2> gpurun_out/bare.err; echo "bench rc=$? wall $((SECONDS-S)) s"
S=$SECONDS; python bench.py --impl reference > gpurun_out/bare_ref.log 2> gpurun_out/bare_ref.err; echo "ref rc=$? wall $((SECONDS-S)) s"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bare.log").read().strip().splitlines()[-1])
print("mine", d["steps"], d["warmup"], d["value"], d["e2e"]["value"], d["clocks"])
d = json.loads(open("gpurun_out/bare_ref.log").read().strip().splitlines()[-1])
print("ref", d["steps"], d["warmup"], d["value"])
PY
