// merge_classic on the device (see merge.cu).
#pragma once

#include <memory>

namespace cobsg {
struct DeviceIndex;
// proj/src/classic_index.cpp:96-115: DataError on differing parameters or
// widths and on duplicate names; UsageError unless both are classic.
std::unique_ptr<DeviceIndex> merge_classic(const DeviceIndex& a, const DeviceIndex& b, int device);
} // namespace cobsg
