# Closing bench after the right-looking panel F: default bench line, smoke.
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02f3_smoke.log 2>&1; tail -1 gpurun_out/r02f3_smoke.log
python bench.py > gpurun_out/r02f3_bench.json 2> gpurun_out/r02f3_bench.err
head -c 300 gpurun_out/r02f3_bench.json; echo
