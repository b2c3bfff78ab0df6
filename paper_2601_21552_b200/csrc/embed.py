"""Embed the device headers as C string literals for NVRTC (build/jit_src.inc)."""
import sys
from pathlib import Path

out, *files = sys.argv[1:]
parts = []
for f in files:
    name = "kSrc_" + Path(f).name.replace(".", "_")
    text = Path(f).read_text()
    chunks = [text[i:i + 12000] for i in range(0, len(text), 12000)] or [""]
    body = "\n".join('R"OOBJIT(' + c + ')OOBJIT"' for c in chunks)
    parts.append(f"static const char {name}[] =\n{body};\n")
Path(out).write_text("".join(parts))
