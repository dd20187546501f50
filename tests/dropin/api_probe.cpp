// Compile-only probe: the drop-in buffer/crc32 headers + the reference's
// engine headers form one program, and the reference's hot-path API is there
// with its exact signatures (buffer.hpp:44-90, cr.hpp:124-206, crc32.hpp:26-34).
#include <type_traits>

#include "gpucrsim/scenario.hpp"

using namespace gpucrsim;

static_assert(std::is_same_v<decltype(&GpuBuffer::chunk_count), uint32_t (GpuBuffer::*)() const>);
static_assert(std::is_same_v<decltype(&GpuBuffer::chunk_bytes), uint64_t (GpuBuffer::*)(uint32_t) const>);
static_assert(std::is_same_v<decltype(&GpuBuffer::content), const std::vector<uint8_t>& (GpuBuffer::*)() const>);
static_assert(std::is_same_v<decltype(&GpuBuffer::read_content),
                             std::vector<uint8_t> (GpuBuffer::*)(uint64_t, uint64_t) const>);
static_assert(std::is_same_v<decltype(&GpuBuffer::write_content),
                             void (GpuBuffer::*)(uint64_t, const uint8_t*, uint64_t)>);
static_assert(std::is_same_v<decltype(&crc32), uint32_t (*)(const void*, size_t)>);
static_assert(std::is_same_v<decltype(&crc32_update), uint32_t (*)(uint32_t, const void*, size_t)>);
static_assert(std::is_base_of_v<CrHooks, CrEngine>);
static_assert(std::is_constructible_v<CrEngine, GpuProcess&>);
static_assert(std::is_same_v<decltype(&CrEngine::checkpoint),
                             void (CrEngine::*)(CrMode, CheckpointTarget, std::function<void(CheckpointImage)>, bool)>);
