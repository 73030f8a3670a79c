"""Print the SASS of one kernel (substring match on the mangled name) from a
cuobjdump -sass dump: python tools/sass_fn.py DUMP NAME_SUBSTR"""
import sys
out, on = [], False
for line in open(sys.argv[1]):
    if "Function :" in line:
        on = sys.argv[2] == line.split("Function :")[1].strip()
    if on:
        out.append(line.rstrip())
print("\n".join(out))
