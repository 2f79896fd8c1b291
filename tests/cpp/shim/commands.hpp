// TEST INFRASTRUCTURE: stand-in for the reference's tools/commands.hpp, so the
// reference's acceptance harness (tests/acceptance.cpp) compiles unmodified.
// cbct::cli::run drives THIS library's CLI (python -m paper_2110_09841_b200,
// the commands.cpp subcommands / flags / CSV formats) in a child process.
#pragma once

namespace cbct::cli {

int run(int argc, const char* const* argv);

}  // namespace cbct::cli
