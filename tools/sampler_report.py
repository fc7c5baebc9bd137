"""Resolve tools/sampler.c output into self / inclusive function tables.
usage: python tools/sampler_report.py gpurun_out/samples.txt [top]"""
import collections
import os
import subprocess
import sys


def resolve(entries):
    """{(module, off)} -> function name, via addr2line per module (local paths
    are remapped from the GPU box's scratch copy to this repo)."""
    by_mod = collections.defaultdict(set)
    for m, o in entries:
        by_mod[m].add(o)
    names = {}
    for m, offs in by_mod.items():
        local = m
        if "/repo/" in m:
            local = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), m.split("/repo/", 1)[1])
        offs = sorted(offs)
        if not os.path.exists(local):
            for o in offs:
                names[(m, o)] = f"{os.path.basename(m)}+{o}"
            continue
        out = subprocess.run(["addr2line", "-f", "-C", "-e", local] + offs, capture_output=True, text=True).stdout
        lines = out.splitlines()
        for i, o in enumerate(offs):
            fn = lines[2 * i] if 2 * i < len(lines) else "??"
            if fn == "??":
                fn = f"{os.path.basename(m)}+{o}"
            names[(m, o)] = fn[:110]
    return names


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    stacks = []
    for ln in open(path):
        if ln.startswith("#") or not ln.strip():
            continue
        fr = []
        for e in ln.strip().split(";"):
            m, _, o = e.rpartition("+")
            fr.append((m, o))
        stacks.append(fr)
    names = resolve({f for s in stacks for f in s})
    n = len(stacks)
    self_c, incl = collections.Counter(), collections.Counter()
    for s in stacks:
        fn = [names[f] for f in s]
        self_c[fn[0]] += 1
        for x in set(fn):
            incl[x] += 1
    print(f"{n} samples")
    print("--- self")
    for k, v in self_c.most_common(top):
        print(f"{100 * v / n:6.2f}%  {k}")
    print("--- inclusive")
    for k, v in incl.most_common(top):
        print(f"{100 * v / n:6.2f}%  {k}")


if __name__ == "__main__":
    main()
