"""Reference CPU arm with shared vs private inputs per replica (cfg5)."""
import sys, os
sys.path.insert(0, os.getcwd())
import bench
for priv in (False, True, False, True):
    g, t, th, tgt, p = bench.run_reference_cpu("cfg5", 3, 1, private=priv)
    print(f"private={p} threads={th}: {g:.1f} GB/s steps {[round(x,3) for x in t]}", flush=True)
print("mem avail GB", bench._mem_available()/1e9)
