"""List backward-branch loops of each transport_kernel instance in a cuobjdump -sass dump
(size, and whether the range holds VOTE / CALL) -- to compare walk-loop code between builds."""
import re, sys
txt = open(sys.argv[1]).read().split("Function : ")
for fn in txt[1:]:
    name = fn.split("\n", 1)[0].strip()
    if "transport_kernel" not in name:
        continue
    ins = re.findall(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", fn)
    addr = [int(a, 16) for a, _ in ins]
    loops = []
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", t)
        m2 = re.search(r"BRA .*`\(\.L_x_(\d+)\)", t)
        tgt = None
        m3 = re.search(r"BRA[^`]*0x([0-9a-f]+)", t)
        if m3:
            tgt = int(m3.group(1), 16)
        if tgt is not None and tgt < int(a, 16):
            body = [x for (b, x) in ins if tgt <= int(b, 16) <= int(a, 16)]
            n = len(body)
            vote = sum("VOTE" in x for x in body)
            call = sum("CALL" in x for x in body)
            loops.append((n, tgt, int(a, 16), vote, call))
    print(name, "instrs", len(ins))
    for n, t, a, v, c in sorted(loops, key=lambda x: x[1]):
        if v and n < 400:
            print(f"   loop {t:#x}-{a:#x} n={n} vote={v} call={c}")
