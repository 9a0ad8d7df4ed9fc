mkdir -p gpurun_out
for t in ${1:-6}; do
  DHSA_COPY_THREADS=$t timeout 600 python tools/host_feed_probe.py > gpurun_out/feed_probe_t$t.json 2> gpurun_out/feed_probe_t$t.err
  echo "== copy threads $t"; cat gpurun_out/feed_probe_t$t.err | tail -24
done
