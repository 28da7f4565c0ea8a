"""Run one config with the layer-kernel event trace of layer k (needs the -DPL_WS_TRACE_ENABLE
variant library via PL_NATIVE_LIB and PL_WS_TRACE=<file> PL_WS_TRACE_K=<k>)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
a = configs.generate(sys.argv[1])[0]
pl.store_zechin_permanent(a)
pl.store_zechin_permanent(a)
