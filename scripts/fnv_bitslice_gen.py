"""Generator + model for the bit-sliced low-byte chain of FNV-1a (multiplier byte 0xb3)."""
C = 0xb3
MULT_BITS = [m for m in range(8) if (C >> m) & 1]   # 0,1,4,5,7

def gen_network():
    """Straight-line ops.  Variables: X{j} (known after plane j resolves).  Emits per column j the
    code computing G{j} from lower X planes and carries; then 'K{j}' = X{j} & G{j} is pushed to column j+1."""
    cols = [[] for _ in range(9)]
    code = {}
    tmp = [0]
    def new():
        tmp[0] += 1
        return f"t{tmp[0]}"
    for j in range(8):
        lines = []
        ins = list(cols[j])
        for m in MULT_BITS:
            if m != 0 and j - m >= 0:
                ins.append(f"X{j-m}")
        # reduce to one plane
        while len(ins) > 1:
            if len(ins) >= 3:
                a, b, c = ins[:3]; ins = ins[3:]
                s, cy = new(), new()
                lines.append(f"const uint32_t {s} = {a} ^ {b} ^ {c};")
                if j + 1 < 8:
                    lines.append(f"const uint32_t {cy} = ({a} & {b}) | ({c} & ({a} ^ {b}));")
                    cols[j+1].append(cy)
                ins.append(s)
            else:
                a, b = ins; ins = []
                s, cy = new(), new()
                lines.append(f"const uint32_t {s} = {a} ^ {b};")
                if j + 1 < 8:
                    lines.append(f"const uint32_t {cy} = {a} & {b};")
                    cols[j+1].append(cy)
                ins.append(s)
        g = ins[0] if ins else "0u"
        lines.append(f"const uint32_t G{j} = {g};")
        code[j] = lines
        if j + 1 < 8:
            cols[j+1].append(f"K{j}")   # X{j} & G{j}, defined by the caller after X{j} resolves
    return code

if __name__ == "__main__":
    code = gen_network()
    n = sum(len(v) for v in code.values())
    for j in range(8):
        print(f"// column {j}")
        for l in code[j]: print(l)
    print("// ops:", n)
