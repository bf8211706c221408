// double log-domain instantiations of the persistent kernel.
#include "fs1_persist_inst.cuh"

namespace fs1 {
static const PersistEntry kTable[] = {
    FS1_PERSIST_ENTRY(double, 1, 4, 1, true),
    FS1_PERSIST_ENTRY(double, 1, 4, 2, true),
    FS1_PERSIST_ENTRY(double, 1, 4, 4, true),
    FS1_PERSIST_ENTRY(double, 1, 4, 8, true),
    FS1_PERSIST_ENTRY(double, 1, 8, 16, true),
    FS1_PERSIST_ENTRY(double, 1, 16, 16, true),
    FS1_PERSIST_ENTRY(double, 1, 4, 16, true),
    FS1_PERSIST_ENTRY(double, 1, 4, 32, true),
    FS1_PERSIST_ENTRY(double, 1, 8, 32, true),
    // short chunks for large c = h/eps (warp span 32 E c <= 650)
    FS1_PERSIST_ENTRY(double, 1, 2, 4, true),
    FS1_PERSIST_ENTRY(double, 1, 2, 8, true),
    FS1_PERSIST_ENTRY(double, 1, 2, 16, true),
    FS1_PERSIST_ENTRY(double, 1, 2, 32, true),
};
const PersistEntry* persist_table_f64l(int* count) {
  *count = (int)(sizeof(kTable) / sizeof(kTable[0]));
  return kTable;
}
}  // namespace fs1
