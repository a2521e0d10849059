"""The bench's attention_c2 section alone (Mixtral shape with real GQA attention, B=64, gamma=4)."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

a = bench.args_parse()
print(json.dumps(bench.section_shape(a, 0, "c2", a.batch, a.n_draft, bench.peaks(), attention=True)))
