// TEST INFRASTRUCTURE ONLY — a command-line probe of the reference's own
// sources (compiled unmodified) for the parts whose C++ runtime use does not
// mix with a Python process (std::filesystem / std::regex of a statically
// linked libstdc++ inside a ctypes-loaded library): run as a subprocess by
// tests/test_io.py.
//   ref_tools scan <dir>   scan_sequence_dir (sequence.cpp:9-43):
//                          "frames N rgb_only R disparity_only D" then one
//                          "index has_rgb" line per frame
#include <cstdio>
#include <cstring>

#include "voxfuse/io/sequence.hpp"

int main(int argc, char** argv) {
  if (argc == 3 && std::strcmp(argv[1], "scan") == 0) {
    const voxfuse::SequenceScan s = voxfuse::scan_sequence_dir(argv[2]);
    std::printf("frames %zu rgb_only %d disparity_only %d\n", s.frames.size(), s.rgb_only, s.disparity_only);
    for (const auto& f : s.frames) std::printf("%d %d\n", f.index, f.rgb_path.empty() ? 0 : 1);
    return 0;
  }
  std::fprintf(stderr, "usage: ref_tools scan <dir>\n");
  return 2;
}
