// Detached-header raw volumes (io.hpp:57-202, 337-428), host side, plus the
// GPU ingest: planes of the last axis streamed from disk through pinned
// staging buffers into device memory (pread of chunk i+1 overlaps the H2D copy
// of chunk i), so a rank of a z-slab job reads only its own planes. Types:
// the reference's uint8 / float32 / uint32 (label maps) and uint16 (config 3).
// PNG (io.hpp:227-330) needs libpng, which this build does not link.
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "capi_internal.cuh"

namespace sslic_b200 {
namespace {

struct Header {
  int rank = 0;
  int64_t dims[kMaxRank] = {1, 1, 1, 1};
  int channels = 1;
  std::string type, endian = "little", data_file;
};

std::string trim(const std::string& s) {
  const size_t a = s.find_first_not_of(" \t\r\n");
  if (a == std::string::npos) return "";
  return s.substr(a, s.find_last_not_of(" \t\r\n") - a + 1);
}

int esize_of(const std::string& t) {
  if (t == "uint8") return 1;
  if (t == "uint16") return 2;
  if (t == "float32" || t == "uint32") return 4;
  throw Error(SSLIC_EIO_TYPE, "unsupported element type: " + t);
}

int dtype_of(const std::string& t) {
  if (t == "uint8") return SSLIC_U8;
  if (t == "uint16") return SSLIC_U16;
  if (t == "float32") return SSLIC_F32;
  throw Error(SSLIC_EIO_TYPE, "unsupported image element type: " + t);
}

bool is_png(const std::string& p) {
  if (p.size() < 4) return false;
  std::string e = p.substr(p.size() - 4);
  std::transform(e.begin(), e.end(), e.begin(), [](unsigned char c) { return std::tolower(c); });
  return e == ".png";
}

// parse_volume_header (io.hpp:123-190): '#' comments and blank lines skipped,
// "key: value" lines, unknown keys ignored; dimension, sizes, type and data
// file are required; little endian only.
Header parse_header(const std::string& path) {
  if (is_png(path)) throw Error(SSLIC_EIO_TYPE, "PNG volumes need libpng (not in this build)");
  std::ifstream f(path);
  if (!f) throw Error(SSLIC_EIO_NOT_FOUND, "cannot open " + path);
  Header h;
  bool saw_dim = false, saw_sizes = false, saw_type = false, saw_data = false;
  std::vector<int64_t> sizes;
  auto to_int = [](const std::string& v, const char* key) {
    try {
      size_t used = 0;
      const int x = std::stoi(v, &used);
      return x;
    } catch (const std::exception&) {
      throw Error(SSLIC_EIO_HEADER, std::string("non-numeric ") + key + ": " + v);
    }
  };
  std::string line;
  while (std::getline(f, line)) {
    line = trim(line);
    if (line.empty() || line[0] == '#') continue;
    const size_t colon = line.find(':');
    if (colon == std::string::npos) throw Error(SSLIC_EIO_HEADER, "header line without ':': " + line);
    const std::string key = trim(line.substr(0, colon)), value = trim(line.substr(colon + 1));
    if (key == "dimension") {
      saw_dim = true;
      h.rank = to_int(value, "dimension");
      if (h.rank < 1 || h.rank > kMaxRank)
        throw Error(SSLIC_EIO_HEADER, "dimension outside [1," + std::to_string(kMaxRank) + "]: " + value);
    } else if (key == "sizes") {
      saw_sizes = true;
      sizes.clear();
      std::istringstream vs(value);
      int64_t v;
      while (vs >> v) sizes.push_back(v);
    } else if (key == "channels") {
      h.channels = to_int(value, "channels");
    } else if (key == "type") {
      saw_type = true;
      h.type = value;
    } else if (key == "endian") {
      h.endian = value;
    } else if (key == "data file") {
      saw_data = true;
      h.data_file = value;
    }
  }
  if (!saw_dim || !saw_sizes || !saw_type || !saw_data)
    throw Error(SSLIC_EIO_HEADER, "header must contain dimension, sizes, type and data file");
  if ((int)sizes.size() != h.rank)
    throw Error(SSLIC_EIO_HEADER, "sizes entry count does not match dimension");
  for (int a = 0; a < h.rank; ++a) {
    if (sizes[a] < 1) throw Error(SSLIC_EIO_HEADER, "non-positive size");
    h.dims[a] = sizes[a];
  }
  if (h.channels < 1) throw Error(SSLIC_EIO_HEADER, "channels must be >= 1");
  esize_of(h.type);
  if (h.endian != "little") throw Error(SSLIC_EIO_TYPE, "unsupported endianness: " + h.endian);
  // relative data file names are resolved beside the header (io.hpp:193-195)
  if (!h.data_file.empty() && h.data_file[0] != '/') {
    const size_t slash = path.find_last_of('/');
    if (slash != std::string::npos) h.data_file = path.substr(0, slash + 1) + h.data_file;
  }
  return h;
}

int64_t voxels(const Header& h) {
  int64_t n = 1;
  for (int a = 0; a < h.rank; ++a) n *= h.dims[a];
  return n;
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

// Payload checks (io.hpp:193-201): the data file must hold exactly the bytes
// the header implies.
void open_payload(const Header& h, Fd& fd) {
  fd.fd = ::open(h.data_file.c_str(), O_RDONLY);
  if (fd.fd < 0) throw Error(SSLIC_EIO_NOT_FOUND, "cannot open " + h.data_file);
  const int64_t want = voxels(h) * h.channels * esize_of(h.type);
  const off_t size = ::lseek(fd.fd, 0, SEEK_END);
  if ((int64_t)size != want)
    throw Error(SSLIC_EIO_SIZE, "payload is " + std::to_string((long long)size) +
                                    " bytes, header implies " + std::to_string((long long)want));
}

void pread_all(int fd, void* dst, size_t bytes, int64_t off) {
  char* p = static_cast<char*>(dst);
  while (bytes > 0) {
    const ssize_t r = ::pread(fd, p, bytes, (off_t)off);
    if (r <= 0) {
      if (r < 0 && errno == EINTR) continue;
      throw Error(SSLIC_EIO_SIZE, "short read");
    }
    p += r;
    bytes -= (size_t)r;
    off += r;
  }
}

void write_bytes(const std::string& path, const void* data, size_t bytes) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw Error(SSLIC_EIO_WRITE, "cannot open " + path + " for writing");
  const size_t w = bytes ? std::fwrite(data, 1, bytes, f) : 0;
  const bool ok = std::fclose(f) == 0 && w == bytes;
  if (!ok) throw Error(SSLIC_EIO_WRITE, "short write to " + path);
}

// write_header (io.hpp:204-228); the payload is <stem>.raw beside the header
std::string write_volume_files(const std::string& path, int rank, const int64_t* dims,
                               int channels, const std::string& type, const void* payload,
                               size_t bytes, const std::string& comment) {
  const size_t slash = path.find_last_of('/');
  const std::string dir = slash == std::string::npos ? "" : path.substr(0, slash + 1);
  std::string stem = slash == std::string::npos ? path : path.substr(slash + 1);
  const size_t dot = stem.find_last_of('.');
  if (dot != std::string::npos && dot > 0) stem = stem.substr(0, dot);
  const std::string data_file = stem + ".raw";
  write_bytes(dir + data_file, payload, bytes);
  std::ostringstream os;
  os << "# sslic volume\n";
  if (!comment.empty()) os << "# " << comment << '\n';
  os << "dimension: " << rank << '\n' << "sizes:";
  for (int a = 0; a < rank; ++a) os << ' ' << dims[a];
  os << '\n' << "channels: " << channels << '\n' << "type: " << type << '\n';
  os << "endian: little\n" << "data file: " << data_file << '\n';
  const std::string text = os.str();
  write_bytes(path, text.data(), text.size());
  return data_file;
}

}  // namespace

// write_labels (io.hpp:396-412) with the label count already known (the
// fused final pass computes the max on the device).
void write_labels_counted(const char* path, int rank, const int64_t* dims,
                          const uint32_t* labels, uint64_t count) {
  int64_t n = 1;
  for (int a = 0; a < rank; ++a) n *= dims[a];
  write_volume_files(path, rank, dims, 1, "uint32", labels, (size_t)n * 4,
                     "label count: " + std::to_string((unsigned long long)count));
}

// write_volume(path, mask_label_contour(img, labels)) (io.hpp:432-454,
// 362-392; default type float32) from the image and the contour bitmask of
// the fused final pass: streamed in chunks, boundary voxels zeroed in every
// channel, other values converted as static_cast<float>(double(v)).
void write_contour_f32(const char* path, const sslic_image* img, const uint32_t* boundary) {
  int64_t n = 1;
  for (int a = 0; a < img->rank; ++a) n *= img->dims[a];
  const int ch = img->channels;
  const size_t slash = std::string(path).find_last_of('/');
  const std::string sp(path);
  const std::string dir = slash == std::string::npos ? "" : sp.substr(0, slash + 1);
  std::string stem = slash == std::string::npos ? sp : sp.substr(slash + 1);
  const size_t dot = stem.find_last_of('.');
  if (dot != std::string::npos && dot > 0) stem = stem.substr(0, dot);
  const std::string data_file = stem + ".raw";
  FILE* f = std::fopen((dir + data_file).c_str(), "wb");
  if (!f) throw Error(SSLIC_EIO_WRITE, "cannot open " + dir + data_file + " for writing");
  constexpr int64_t kChunk = (int64_t)1 << 22;
  std::vector<float> buf((size_t)kChunk * ch);
  bool ok = true;
  for (int64_t v0 = 0; v0 < n && ok; v0 += kChunk) {
    const int64_t v1 = std::min(n, v0 + kChunk);
    for (int64_t v = v0; v < v1; ++v) {
      const bool b = boundary[v >> 5] >> (v & 31) & 1u;
      for (int c = 0; c < ch; ++c) {
        const int64_t i = v * ch + c;
        double x;
        switch (img->dtype) {
          case SSLIC_U8: x = static_cast<const uint8_t*>(img->data)[i]; break;
          case SSLIC_U16: x = static_cast<const uint16_t*>(img->data)[i]; break;
          case SSLIC_F32: x = static_cast<const float*>(img->data)[i]; break;
          default: x = static_cast<const double*>(img->data)[i];
        }
        buf[(size_t)((v - v0) * ch + c)] = b ? 0.0f : static_cast<float>(x);
      }
    }
    const size_t cnt = (size_t)((v1 - v0) * ch);
    ok = std::fwrite(buf.data(), sizeof(float), cnt, f) == cnt;
  }
  ok = std::fclose(f) == 0 && ok;
  if (!ok) throw Error(SSLIC_EIO_WRITE, "short write to " + dir + data_file);
  std::ostringstream os;
  os << "# sslic volume\n" << "dimension: " << img->rank << '\n' << "sizes:";
  for (int a = 0; a < img->rank; ++a) os << ' ' << img->dims[a];
  os << '\n' << "channels: " << ch << '\n' << "type: float32\n";
  os << "endian: little\n" << "data file: " << data_file << '\n';
  const std::string text = os.str();
  write_bytes(path, text.data(), text.size());
}

}  // namespace sslic_b200

using namespace sslic_b200;

extern "C" {

int sslic_volume_info_read(const char* path, sslic_volume_info* out) {
  return guarded([&] {
    if (!path || !out) throw Error(SSLIC_EINVAL, "null argument");
    const Header h = parse_header(path);
    out->rank = h.rank;
    for (int a = 0; a < 4; ++a) out->dims[a] = a < h.rank ? h.dims[a] : 1;
    out->channels = h.channels;
    out->label_map = h.type == "uint32";
    out->dtype = out->label_map ? -1 : dtype_of(h.type);
    return SSLIC_OK;
  });
}

int sslic_volume_read(const char* path, int64_t plane_begin, int64_t plane_end, void* dst,
                      int device) {
  return guarded([&] {
    if (!path || !dst) throw Error(SSLIC_EINVAL, "null argument");
    const Header h = parse_header(path);
    const int64_t last = h.dims[h.rank - 1];
    if (plane_begin < 0 || plane_end > last || plane_begin > plane_end)
      throw Error(SSLIC_ERANGE, "plane range outside the volume");
    Fd fd;
    open_payload(h, fd);
    const int64_t plane_bytes = voxels(h) / last * h.channels * esize_of(h.type);
    const int64_t off = plane_begin * plane_bytes;
    const int64_t bytes = (plane_end - plane_begin) * plane_bytes;
    if (device < 0) {
      pread_all(fd.fd, dst, (size_t)bytes, off);
      return SSLIC_OK;
    }
    // disk -> pinned staging (2 x 64 MB) -> device, pread of the next chunk
    // overlapping the copy of the current one
    SSLIC_CUDA_CHECK(cudaSetDevice(device));
    const int64_t chunk = std::min<int64_t>(bytes, 64ll << 20);
    char* stage = nullptr;
    SSLIC_CUDA_CHECK(cudaMallocHost(&stage, (size_t)std::max<int64_t>(chunk, 1) * 2));
    cudaStream_t s = nullptr;
    cudaEvent_t done[2] = {nullptr, nullptr};
    try {
      SSLIC_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      for (auto& e : done) SSLIC_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      int buf = 0;
      for (int64_t pos = 0; pos < bytes; pos += chunk, buf ^= 1) {
        const int64_t len = std::min(chunk, bytes - pos);
        SSLIC_CUDA_CHECK(cudaEventSynchronize(done[buf]));  // staging buffer free again
        pread_all(fd.fd, stage + buf * chunk, (size_t)len, off + pos);
        SSLIC_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(dst) + pos, stage + buf * chunk,
                                         (size_t)len, cudaMemcpyHostToDevice, s));
        SSLIC_CUDA_CHECK(cudaEventRecord(done[buf], s));
      }
      SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));
    } catch (...) {
      if (s) cudaStreamSynchronize(s);
      for (auto& e : done)
        if (e) cudaEventDestroy(e);
      if (s) cudaStreamDestroy(s);
      cudaFreeHost(stage);
      throw;
    }
    for (auto& e : done) cudaEventDestroy(e);
    cudaStreamDestroy(s);
    cudaFreeHost(stage);
    return SSLIC_OK;
  });
}

int sslic_volume_write(const char* path, const sslic_image* img) {
  return guarded([&] {
    if (!path || !img || !img->data) throw Error(SSLIC_EINVAL, "null argument");
    if (is_png(path)) throw Error(SSLIC_EIO_TYPE, "PNG volumes need libpng (not in this build)");
    const char* type = img->dtype == SSLIC_U8    ? "uint8"
                       : img->dtype == SSLIC_U16 ? "uint16"
                       : img->dtype == SSLIC_F32 ? "float32"
                                                 : nullptr;
    if (!type) throw Error(SSLIC_EIO_TYPE, "volumes are stored as uint8, uint16 or float32");
    int64_t n = img->channels;
    for (int a = 0; a < img->rank; ++a) n *= img->dims[a];
    write_volume_files(path, img->rank, img->dims, img->channels, type, img->data,
                       (size_t)n * esize_of(type), "");
    return SSLIC_OK;
  });
}

int sslic_labels_write(const char* path, int rank, const int64_t* dims, const uint32_t* labels) {
  return guarded([&] {
    if (!path || !dims || !labels || rank < 1 || rank > 4)
      throw Error(SSLIC_EINVAL, "bad label map");
    int64_t n = 1;
    for (int a = 0; a < rank; ++a) n *= dims[a];
    uint32_t mx = 0;
    for (int64_t i = 0; i < n; ++i) mx = std::max(mx, labels[i]);
    // write_labels (io.hpp:396-412): uint32, "label count: max + 1" comment
    write_volume_files(path, rank, dims, 1, "uint32", labels, (size_t)n * 4,
                       "label count: " + std::to_string((unsigned long long)mx + 1));
    return SSLIC_OK;
  });
}

int sslic_labels_read(const char* path, uint32_t* labels_out) {
  return guarded([&] {
    if (!path || !labels_out) throw Error(SSLIC_EINVAL, "null argument");
    const Header h = parse_header(path);
    if (h.type != "uint32")
      throw Error(SSLIC_EIO_TYPE, "label maps must have type uint32, got " + h.type);
    if (h.channels != 1) throw Error(SSLIC_EIO_HEADER, "label maps must have a single channel");
    Fd fd;
    open_payload(h, fd);
    pread_all(fd.fd, labels_out, (size_t)voxels(h) * 4, 0);
    return SSLIC_OK;
  });
}

}  // extern "C"
