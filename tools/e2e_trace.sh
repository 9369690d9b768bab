# host-pipeline timelines (BTD_HOST_TRACE=1) for c1 at different chunk widths
for w in 64 32; do
  echo "== c1 minw=$w"
  BTD_HOST_TRACE=1 BTD_HOST_MINW=$w python bench.py --config c1 --steps 2 --warmup 3 --no-cpu --no-check 2>&1 >/dev/null | grep -A9 "btd host" | tail -10
done
