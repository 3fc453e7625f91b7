import re, sys, subprocess, collections
fn = sys.argv[1] if len(sys.argv) > 1 else '_ZN3xsd16transport_kernelILi0ELb1ELb1EEEvNS_15TransportParamsE'
out = subprocess.run(['cuobjdump', '-sass', '-fun', fn, 'paper_2201_13191_b200/build/transport.o'],
                     capture_output=True, text=True).stdout.splitlines()
ins = []
calls = set()
for l in out:
    m = re.match(r'\s*/\*([0-9a-f]+)\*/\s+(.*?);', l)
    if not m:
        continue
    a = int(m.group(1), 16)
    ins.append((a, m.group(2)))
    if 'CALL' in m.group(2):
        mm = re.search(r'(0x[0-9a-f]+)', m.group(2))
        if mm:
            calls.add(int(mm.group(1), 16))
end = ins[-1][0] + 16
pts = [0] + sorted(calls)
for i, t in enumerate(pts):
    nxt = pts[i + 1] if i + 1 < len(pts) else end
    seg = [s for a, s in ins if t <= a < nxt]
    ops = collections.Counter((s.split()[1] if s.startswith('@') else s.split()[0]).split('.')[0] for s in seg)
    print(f"{hex(t):>9} {nxt - t:7d} B  calls_out={sum('CALL' in s for s in seg):3d}  top={ops.most_common(5)}")
