# e2e (host buffers) vs the host pipeline's chunk count, small and large configs
for c in cfg1 cfg3 cfg2; do for k in 1 2 4 8; do
  echo "$c chunks=$k $(CGMIMO_HOST_CHUNKS=$k python tools/e2e_time.py $c 2>&1 | tail -1)"
done; done
