// float log-domain instantiations of the persistent kernel.
#include "fs1_persist_inst.cuh"

namespace fs1 {
static const PersistEntry kTable[] = {
    FS1_PERSIST_ENTRY(float, 0, 8, 1, true),
    FS1_PERSIST_ENTRY(float, 0, 16, 1, true),
    FS1_PERSIST_ENTRY(float, 0, 32, 1, true),
    FS1_PERSIST_ENTRY(float, 0, 64, 1, true),
    FS1_PERSIST_ENTRY(float, 0, 64, 2, true),
    FS1_PERSIST_ENTRY(float, 0, 64, 4, true),
    FS1_PERSIST_ENTRY(float, 0, 32, 2, true),
    FS1_PERSIST_ENTRY(float, 0, 32, 4, true),
    FS1_PERSIST_ENTRY(float, 0, 32, 8, true),
    FS1_PERSIST_ENTRY(float, 0, 32, 16, true),
};
const PersistEntry* persist_table_f32l(int* count) {
  *count = (int)(sizeof(kTable) / sizeof(kTable[0]));
  return kTable;
}
}  // namespace fs1
