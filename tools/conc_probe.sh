cd /root/repo
for k in 1 4 16; do
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/cc.log &
  P=$!
  CONC_CHUNKS=$k tools/sweep_probe conc 30 20
  kill $P
  python3 -c "
import statistics
rows=[l.split(',') for l in open('/tmp/cc.log') if l.strip()]
hot=[(float(a),float(b)) for a,b in rows if float(b)>400]
print(f'   {statistics.median([h[0] for h in hot]):.0f} MHz {statistics.median([h[1] for h in hot]):.0f} W' if hot else 'idle')"
done
