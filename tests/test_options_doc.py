"""Engine options: every name atk_set_option accepts (csrc/api.cu) is documented in
include/atk.h and in INTEGRATION.md's option table, and vice versa (CPU, static)."""
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _accepted():
    src = (ROOT / "paper_2010_10131_b200" / "csrc" / "api.cu").read_text()
    return set(re.findall(r'k == "([a-z_0-9]+)"', src))


def test_header_documents_every_option():
    hdr = (ROOT / "include" / "atk.h").read_text()
    documented = set(re.findall(r'^ \*   "([a-z_0-9]+)"', hdr, flags=re.M))
    assert documented == _accepted()


def test_integration_table_lists_engine_options():
    doc = (ROOT / "INTEGRATION.md").read_text()
    listed = set(re.findall(r'^\| `([a-z_0-9]+)` \|', doc, flags=re.M))
    missing = _accepted() - listed
    # the table may also list other backticked keys; every engine option must be there
    assert not missing, f"options missing from INTEGRATION.md: {sorted(missing)}"
