// Drop-in replacement for the reference's src/io.cpp on top of the C ABI in
// include/vk_io.h.
//
// voxelkit::io::read_volume / write_volume (reference include/voxelkit/io.hpp,
// src/io.cpp:53-158) keep their signatures, exception types and messages; the
// NDIV parsing and the byte-identical header writer live in
// csrc/vk_io.cpp.  Link this TU instead of src/io.cpp (it needs no JSON
// library).  export_slice (io.cpp:160-196, the CLI's `export-slice`, outside
// the deconvolution path) is restated here so the TU replaces io.cpp whole.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <string>
#include <vector>

#include "voxelkit/errors.hpp"
#include "voxelkit/image.hpp"
#include "voxelkit/io.hpp"
#include "vk_io.h"

namespace voxelkit::io {

namespace {

std::string strip(const std::string& m, const char* name) {
  const std::string p = std::string(name) + ": ";
  return m.rfind(p, 0) == 0 ? m.substr(p.size()) : m;
}

[[noreturn]] void rethrow(vk_status st) {
  const std::string m = vk_last_error();
  switch (st) {
    case VK_ERR_BAD_MAGIC: throw BadMagic(strip(m, "BadMagic"));
    case VK_ERR_HEADER_MISMATCH: throw HeaderMismatch(strip(m, "HeaderMismatch"));
    case VK_ERR_TRUNCATED: throw TruncatedPayload(strip(m, "TruncatedPayload"));
    case VK_ERR_SHAPE: throw ShapeMismatch(strip(m, "ShapeMismatch"));
    default: throw Error(m);
  }
}

int to_vk(Elem e) {
  switch (e) {
    case Elem::f32: return VK_ELEM_F32;
    case Elem::u16: return VK_ELEM_U16;
    case Elem::u32_label: return VK_ELEM_U32;
    case Elem::boolean: return VK_ELEM_BOOL;
  }
  return VK_ELEM_F32;
}

const void* raw(const NdImage& img) {
  switch (img.elem()) {
    case Elem::f32: return img.values<float>().data();
    case Elem::u16: return img.values<std::uint16_t>().data();
    case Elem::u32_label: return img.values<std::uint32_t>().data();
    case Elem::boolean: return img.values<std::uint8_t>().data();
  }
  return nullptr;
}

template <class T>
std::vector<T> payload(const std::string& path, vk_volume_info& info) {
  std::uint64_t n = 1;
  for (int a = 0; a < info.rank; ++a) n *= info.shape[a];
  std::vector<T> v(n);
  const vk_status st = vk_volume_read(path.c_str(), &info, v.data(), n * sizeof(T));
  if (st != VK_OK) rethrow(st);
  return v;
}

}  // namespace

void write_volume(const std::string& path, const NdImage& img) {
  if (img.rank() < 1 || img.rank() > VK_VOLUME_MAX_RANK)  // io.cpp:33-41 (axes_for_rank)
    throw HeaderMismatch("unsupported rank " + std::to_string(img.rank()));
  vk_volume_info info{};
  info.elem = to_vk(img.elem());
  info.rank = static_cast<int>(img.rank());
  for (int a = 0; a < info.rank; ++a) info.shape[a] = img.shape()[a];
  if (img.spacing() && img.spacing()->size() == img.rank()) {
    info.has_spacing = 1;
    for (int a = 0; a < info.rank; ++a) info.spacing[a] = (*img.spacing())[a];
  }
  const vk_status st = vk_volume_write(path.c_str(), &info, raw(img));
  if (st != VK_OK) rethrow(st);
}

NdImage read_volume(const std::string& path) {
  vk_volume_info info{};
  const vk_status st = vk_volume_info_read(path.c_str(), &info);  // every header / length check
  if (st != VK_OK) rethrow(st);
  const Shape shape(info.shape, info.shape + info.rank);
  NdImage img;
  switch (info.elem) {
    case VK_ELEM_F32: img = NdImage::f32(shape, payload<float>(path, info)); break;
    case VK_ELEM_U16: img = NdImage::u16(shape, payload<std::uint16_t>(path, info)); break;
    case VK_ELEM_U32: img = NdImage::labels(shape, payload<std::uint32_t>(path, info)); break;
    default: img = NdImage::boolean(shape, payload<std::uint8_t>(path, info)); break;
  }
  if (info.has_spacing) img = img.with_spacing(std::vector<double>(info.spacing, info.spacing + info.rank));
  return img;
}

void export_slice(const NdImage& img, std::size_t axis, std::size_t index, const std::string& path) {
  if (img.rank() != 3) throw ShapeMismatch("export_slice expects a 3D volume");
  if (axis > 2) throw Error("axis must be 0, 1 or 2");
  if (index >= img.extent(axis)) throw Error("slice index out of range");
  const NdImage f = img.as_f32();
  const auto v = f.f32_values();
  const auto st = f.strides();
  // the two remaining axes, in order: rows = first, columns = second
  const std::size_t ra = axis == 0 ? 1 : 0, ca = axis == 2 ? 1 : 2;
  const std::size_t rows = f.extent(ra), cols = f.extent(ca);
  std::vector<float> px(rows * cols);
  float lo = std::numeric_limits<float>::max(), hi = std::numeric_limits<float>::lowest();
  for (std::size_t r = 0; r < rows; ++r)
    for (std::size_t c = 0; c < cols; ++c) {
      const float x = v[index * st[axis] + r * st[ra] + c * st[ca]];
      px[r * cols + c] = x;
      lo = std::min(lo, x);
      hi = std::max(hi, x);
    }
  std::ofstream out(path, std::ios::binary);
  if (!out) throw Error("cannot open '" + path + "' for writing");
  out << "P5\n" << cols << " " << rows << "\n255\n";
  const double k = hi > lo ? 255.0 / (hi - lo) : 0.0;
  for (float x : px) out.put(static_cast<char>(std::clamp(static_cast<int>((x - lo) * k + 0.5), 0, 255)));
  if (!out) throw Error("write to '" + path + "' failed");
}

}  // namespace voxelkit::io
