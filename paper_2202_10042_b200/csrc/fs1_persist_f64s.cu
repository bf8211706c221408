// double scaling-domain instantiations of the persistent kernel.
#include "fs1_persist_inst.cuh"

namespace fs1 {
static const PersistEntry kTable[] = {
    FS1_PERSIST_ENTRY(double, 1, 4, 1, false),
    FS1_PERSIST_ENTRY(double, 1, 4, 2, false),
    FS1_PERSIST_ENTRY(double, 1, 4, 4, false),
    FS1_PERSIST_ENTRY(double, 1, 4, 8, false),
    FS1_PERSIST_ENTRY(double, 1, 4, 16, false),
    FS1_PERSIST_ENTRY(double, 1, 8, 4, false),
    FS1_PERSIST_ENTRY(double, 1, 8, 16, false),
    FS1_PERSIST_ENTRY(double, 1, 16, 16, false),
};
const PersistEntry* persist_table_f64s(int* count) {
  *count = (int)(sizeof(kTable) / sizeof(kTable[0]));
  return kTable;
}
}  // namespace fs1
