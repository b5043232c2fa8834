"""The README's Python usage example, run as written (documentation check):
the first ```python block of README.md is extracted and executed."""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.chdir(ROOT)

text = open(os.path.join(ROOT, "README.md")).read()
block = re.search(r"```python\n(.*?)```", text, re.S).group(1)
scope = {}
exec(compile(block, "README.md", "exec"), scope)
import torch  # noqa: E402

torch.cuda.synchronize()
print("readme snippet ok", scope["y"].shape, scope["y2"].shape, scope["hout"].shape, scope["mid"].shape,
      "d3 variant", scope["d3"].launch_info(2, 3)["variant"])
