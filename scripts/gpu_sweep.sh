timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout -k 10 900 python bench.py --sweep --sweep-csv gpurun_out/sweep.csv > gpurun_out/sweep.json 2> gpurun_out/sweep.err
