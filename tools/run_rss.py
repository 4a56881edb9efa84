"""Run a command, then print its wall time and the peak RSS of the child (dev tool)."""
import resource, subprocess, sys, time
t0 = time.time()
rc = subprocess.call(sys.argv[1:])
ru = resource.getrusage(resource.RUSAGE_CHILDREN)
print(f"rc {rc} wall {time.time() - t0:.1f}s maxrss {ru.ru_maxrss / 1e6:.2f} GB", flush=True)
