// TEST INFRASTRUCTURE: cbct::cli::run for the reference's acceptance harness
// (criterion 7) — execs `python3 -m paper_2110_09841_b200 <args>` with the
// repository root (CBCT_B200_ROOT, else the compile-time root) on PYTHONPATH.
#include <sys/wait.h>
#include <unistd.h>

#include <cstdlib>
#include <string>
#include <vector>

#include "commands.hpp"

#ifndef CBCT_B200_ROOT_DEFAULT
#define CBCT_B200_ROOT_DEFAULT "."
#endif

namespace cbct::cli {

int run(int argc, const char* const* argv) {
    const char* root = std::getenv("CBCT_B200_ROOT");
    std::string r = root ? root : CBCT_B200_ROOT_DEFAULT;
    const char* py = std::getenv("PYTHON");
    std::vector<std::string> args = {py ? py : "python3", "-m", "paper_2110_09841_b200"};
    for (int i = 1; i < argc; ++i) args.emplace_back(argv[i]);
    pid_t pid = fork();
    if (pid < 0) return 1;
    if (pid == 0) {
        const char* old = std::getenv("PYTHONPATH");
        std::string pp = r + (old ? ":" + std::string(old) : "");
        setenv("PYTHONPATH", pp.c_str(), 1);
        std::vector<char*> cargv;
        for (auto& a : args) cargv.push_back(a.data());
        cargv.push_back(nullptr);
        execvp(cargv[0], cargv.data());
        _exit(127);
    }
    int status = 0;
    if (waitpid(pid, &status, 0) < 0) return 1;
    return WIFEXITED(status) ? WEXITSTATUS(status) : 1;
}

}  // namespace cbct::cli
