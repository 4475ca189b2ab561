"""Counts SASS opcodes of one kernel in the built library.
  python tools/sass_count.py <name-substring> [opcode ...] [--lib path]"""
import re
import subprocess
import sys

args = sys.argv[1:]
lib = "paper_2511_21669_b200/libdsdsim.so"
if "--lib" in args:
    i = args.index("--lib")
    lib = args[i + 1]
    del args[i:i + 2]
name, ops = args[0], args[1:]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in out.split("Function : ")[1:]:
    fname = f.split("\n", 1)[0].strip()
    if name not in fname:
        continue
    ins = re.findall(r"/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", f)
    counts = {o: sum(1 for x in ins if x.split(".")[0] == o) for o in ops}
    print(fname, len(ins), counts)
