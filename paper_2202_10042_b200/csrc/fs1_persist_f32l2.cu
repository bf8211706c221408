// float log-domain instantiations of the persistent kernel.
#include "fs1_persist_inst.cuh"

namespace fs1 {
static const PersistEntry kTable[] = {
    FS1_PERSIST_ENTRY(float, 0, 16, 2, true),
    FS1_PERSIST_ENTRY(float, 0, 16, 4, true),
    FS1_PERSIST_ENTRY(float, 0, 16, 8, true),
    FS1_PERSIST_ENTRY(float, 0, 16, 16, true),
    FS1_PERSIST_ENTRY(float, 0, 16, 32, true),
    FS1_PERSIST_ENTRY(float, 0, 8, 2, true),
    FS1_PERSIST_ENTRY(float, 0, 8, 4, true),
    FS1_PERSIST_ENTRY(float, 0, 8, 8, true),
    FS1_PERSIST_ENTRY(float, 0, 8, 16, true),
    FS1_PERSIST_ENTRY(float, 0, 8, 32, true),
    FS1_PERSIST_ENTRY(float, 0, 4, 1, true),
    FS1_PERSIST_ENTRY(float, 0, 4, 2, true),
    FS1_PERSIST_ENTRY(float, 0, 4, 4, true),
    FS1_PERSIST_ENTRY(float, 0, 4, 8, true),
    FS1_PERSIST_ENTRY(float, 0, 4, 16, true),
    FS1_PERSIST_ENTRY(float, 0, 4, 32, true),
};
const PersistEntry* persist_table_f32l2(int* count) {
  *count = (int)(sizeof(kTable) / sizeof(kTable[0]));
  return kTable;
}
}  // namespace fs1
