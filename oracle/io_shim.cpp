// TEST INFRASTRUCTURE ONLY. Stand-in for the reference's libpng-based image
// I/O (src/image_io.cpp; libpng is not in this image) so that dataset.cpp —
// the reference's own write_disparity_png quantisation and write_boxes — can
// be compiled in place for the export fixtures (tests/golden/make_golden_export.py).
// The writers record the image they are handed instead of encoding it; the
// readers are unavailable.
#include <cstdint>
#include <stdexcept>
#include <string>

#include "tsgm/image_io.hpp"

namespace tsgm_shim {
tsgm::Image<std::uint16_t> last16;
tsgm::GrayImage last8;
std::string last_path;
}  // namespace tsgm_shim

namespace tsgm::io {

GrayImage read_gray(const std::string& path) {
    throw std::runtime_error("io shim: read_gray unavailable (" + path + ")");
}
Image<std::uint16_t> read_gray16_png(const std::string& path) {
    throw std::runtime_error("io shim: read_gray16_png unavailable (" + path + ")");
}
void write_gray_png(const std::string& path, const GrayImage& img) {
    tsgm_shim::last8 = img;
    tsgm_shim::last_path = path;
}
void write_gray16_png(const std::string& path, const Image<std::uint16_t>& img) {
    tsgm_shim::last16 = img;
    tsgm_shim::last_path = path;
}

}  // namespace tsgm::io
