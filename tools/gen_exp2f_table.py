"""Print glibc's __exp2f_data.tab (EXP2F_TABLE_BITS = 5) to correct rounding:
tab[i] = asuint64(2^(i/32)) - (i << 47).  Used for csrc/expf_glibc.h."""
import struct
from decimal import Decimal, getcontext

getcontext().prec = 60
for i in range(32):
    v = (Decimal(i) / 32 * Decimal(2).ln()).exp()
    b = struct.unpack("<Q", struct.pack("<d", float(format(v, ".40e"))))[0]
    print("0x%016xULL," % ((b - (i << 47)) & (2**64 - 1)))
