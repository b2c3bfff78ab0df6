"""Aggregate tools/host_profile.sh samples: leaf frame (function, line) counts
over the threads doing work (sleeping pool workers are dropped)."""
import collections
import re
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/host_samples.txt"
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 1
leaf, incl = collections.Counter(), collections.Counter()
threads = re.split(r"^Thread .*$", open(path).read(), flags=re.M)


def name(line):
    line = re.sub(r"^#\d+\s+(0x[0-9a-f]+ in )?", "", line).replace("(anonymous namespace)::", "")
    m = re.search(r" at (\S+):(\d+)", line)
    fn = line.split("(")[0].strip()
    return f"{fn} @{m.group(1).split('/')[-1]}:{m.group(2)}" if m else fn


n = 0
for t in threads:
    fr = [ln for ln in t.strip().split("\n") if ln.startswith("#")]
    if not fr or any(w in fr[0] for w in ("pthread_cond_wait", "futex", "__GI___poll", "epoll", "nanosleep")) \
            or re.search(r"in \?\? \(\) from /lib/x86_64-linux-gnu/libc", fr[0]):
        continue
    if not any("libscuba_oob" in f or " at " in f for f in fr):
        continue
    n += 1
    leaf[" < ".join(name(f) for f in fr[:depth])] += 1
    for f in set(name(f).split(" @")[0] for f in fr):
        incl[f] += 1
print(f"{n} busy thread samples")
for k, v in leaf.most_common(45):
    print(f"{v:5d} {100 * v / n:5.1f}%  {k[:200]}")
print("--- inclusive (function)")
for k, v in incl.most_common(25):
    print(f"{v:5d} {100 * v / n:5.1f}%  {k[:150]}")
