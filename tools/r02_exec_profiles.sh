# Executor / K2 measurements after the K2 rework (round 2): timing table, traces, MLE, K2 strip traces.
cp ab/libexageo_cur.so paper_1708_02835_b200/_lib/libexageo.so
python tools/tile_tasks_timing.py 400 800 1200 1600 2000 2400 2800 3200 3600 4000 > gpurun_out/r02_exec_timing.txt 2>&1
python tools/tile_task_trace.py 1600 > gpurun_out/r02_exec_trace_n1600.txt 2>&1
python tools/tile_task_trace.py 400 > gpurun_out/r02_exec_trace_n400.txt 2>&1
python tools/mle_graph_timing.py > gpurun_out/r02_exec_mle.txt 2>&1
./tools/potrf_bench_trace > gpurun_out/r02_k2_isolated.txt 2>&1
cp ab/libexageo_trace.so paper_1708_02835_b200/_lib/libexageo.so
python tools/chain_k2_trace.py 1600 > gpurun_out/r02_k2_chain.txt 2>&1
cp ab/libexageo_cur.so paper_1708_02835_b200/_lib/libexageo.so
