# bulk peer copies: parity tests, step time with 0/1/7 stand-in peers, ncu instruction counts 0 vs 7 peers
timeout 600 python -m pytest tests/test_gpu_fast.py -q -k "peer" 2>&1 | tail -2
for n in 0 1 7; do timeout 300 python tools/peer_probe.py $n; done
LOPT_PEER_SCALAR=1 timeout 300 python tools/peer_probe.py 7
for n in 0 7; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"apply_pair" -s 3 -c 1 -o gpurun_out/prof_peers$n python tools/peer_probe.py $n 2 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/prof_peers$n.ncu-rep > gpurun_out/prof_peers${n}_summary.txt 2>&1
  grep -E "Duration|warp instructions|DRAM Throughput" gpurun_out/prof_peers${n}_summary.txt
done
